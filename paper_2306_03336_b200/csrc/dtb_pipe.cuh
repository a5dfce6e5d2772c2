// dtb_pipe.cuh — the pipelined (2.5-D) streaming kernel and its launcher
// (instantiated per element type by dtb_pipe_f64.cu / dtb_pipe_f32.cu).
//
// Temporal blocking by a warp pipeline instead of a tile-wide sweep: a
// "pipeline" is S warps; warp s advances rows from time level 2s to 2s+2 and
// hands them to warp s+1 through a small shared-memory ring, so the h = 2S
// fused steps of a pass flow through the pipeline while it marches down a
// tall column strip ("segment") of the domain:
//
//   HBM --cp.async--> ring0 -> [warp 0: t -> t+2] -> ring1 -> [warp 1] -> ...
//                              -> [warp S-1: t+h-2 -> t+h] --STG--> HBM
//
// Each warp streams its rows through two Levels of the running-sum form
// (dtb_core.cuh): an arriving row finishes the row above it at level 1, whose
// output finishes the row above that at level 2. There are no band seams, no
// CTA-wide barriers and no pre-read halo registers; y-redundancy exists only
// at segment ends (segments are hundreds to thousands of rows) and the HBM
// traffic of a pass is one read + one write of every owned cell, overlapped
// with the FP work by the ring prefetch. Each warp spans the strip width
// (32*K columns, lane-owned K-column chunks, shuffles for W/E); every update
// is the reference's FMA-free W,E,S,C,N expression (kernel.py:137-139), so
// results stay bitwise equal to jacobi_reference.
//
// Synchronisation inside a pipeline is by monotonic row counters in shared
// memory (st.release.cta / ld.acquire.cta): prod[s] = rows written into ring
// s, cons[s] = rows ring s's reader no longer needs.
#pragma once
#include <algorithm>
#include <cstring>
#include <type_traits>

#include "dtb_internal.h"
#include "dtb_tile_io.cuh"

#ifndef DTB_PIPE_PROBE
#define DTB_PIPE_PROBE 0  // debug builds: per-stage wait-cycle counters (dtb_debug_pipe_probe)
#endif

namespace dtb {

constexpr int kPipeStages = 4;   // stage warps per pipeline (2 steps each): h = 8

#if DTB_PIPE_PROBE
__device__ unsigned long long g_pipe_probe[8][3];
#endif

__device__ __forceinline__ void pipe_cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void pipe_cp_async(uint32_t dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void pipe_cp_async(uint32_t dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
// 16-byte global stores of a lane's 4-element fp64 row chunk, predicated (no
// branch): the last stage's owned-row store in the steady loop. No "memory"
// clobber: nothing in the kernel reads the destination, and the clobber would
// pin the next rows' shared loads behind the store.
__device__ __forceinline__ void st_row_pred(bool p, double* g, const double (&v)[4]) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0;\n"
               " @q st.global.v2.f64 [%1], {%2, %3};\n"
               " @q st.global.v2.f64 [%1+16], {%4, %5}; }"
               ::"r"((unsigned)p), "l"(g), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]));
}

template <int N>
__device__ __forceinline__ void pipe_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void pipe_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

// Ring geometry (rows of 32*K elements, the tile row layout incl. swizzle).
// fp64 rows need a deeper HBM prefetch than fp32 rows (same 1 KB per row, half
// the cells, so half the compute per row to hide a row's latency behind).
template <typename T>
struct PipeCfg {
  // lane width and warps per CTA: a 1 KB row per warp-row, 16 warps = 4
  // pipelines, one per SM sub-partition (fp64 K=8 x 8 warps, 2 KB rows, fewer
  // shuffles and selects per cell, measured 11 % slower on C4: two warps per
  // sub-partition leave the FP64 latency exposed)
  static constexpr int kK = sizeof(T) == 8 ? 4 : 8;
  static constexpr int kWarps = 16;
  static constexpr bool kDeep = sizeof(T) == 8;
  static constexpr int kRing0Rows = kDeep ? 16 : 12;  // stage 0's HBM prefetch ring
  static constexpr int kRingRows = 12;                // ring between stages
  static constexpr int kPrefetch = kDeep ? 10 : 6;    // HBM rows in flight per pipeline
};

struct PipeTile {
  int Lw, Lh;        // load region (tile-local rows/cols)
  int gx0, gy0;      // padded global coords of tile (0,0)
  int ox0, ox1;      // store columns (owned, + ghost at domain edges), tile-local
  int oy0, oy1;      // store rows, tile-local
  int qy0, qy1;      // owned rows, tile-local (oy before a HaloMirror store window)
  bool vec;          // global side 16-byte aligned per chunk
  int xl, xr;        // columns exact after the pass: [xl, xr) (the pass's steps
                     // in from every halo side; domain ghost columns are frozen)
};

// One pipeline stage warp advancing one tile (segment) by `levels` (0, 1 or
// 2) steps. seq0: the pipeline-wide row sequence number of this tile's row 0
// (ring slot = seq % ring rows). `src` is read only by stage 0; `dst` written
// only by the last stage. Rows 0 and Lh-1 are the frozen frame.
template <typename T, int K, bool SYM, bool DYN, bool MIR>
__device__ __forceinline__ void pipe_stage(const PipeTile& pt, int stage, int nstages, int levels,
                                           int seq0, const T* __restrict__ src,
                                           T* __restrict__ dst, int64_t pitch, uint32_t ring_in,
                                           uint32_t ring_out, int* prod, int* cons,
                                           const Weights<T>& wt, const LaneCtx& lc,
                                           const HaloMirror<T>* mir) {
  typedef Tile<T, K> L;
  typedef Level<T, K, SYM, DYN> Lv;
  constexpr int E = L::EPC, CH = L::CH;
  constexpr uint32_t RB = (uint32_t)(L::ROW * sizeof(T));  // bytes per ring row
  constexpr int kRing0Rows = PipeCfg<T>::kRing0Rows, kRingRows = PipeCfg<T>::kRingRows,
                kPrefetch = PipeCfg<T>::kPrefetch;
  constexpr int kSleep = 400;  // ns between ring-counter polls
  const int lane = lc.lane;
  const int Lh = pt.Lh;
  uint32_t off[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) off[j] = (uint32_t)(L::swz(lane * CH + j) * 16);
  const bool first = stage == 0;
  const bool lastst = stage == nstages - 1;
#if DTB_PIPE_PROBE
  unsigned long long w_in = 0, w_out = 0, t_all = clock64();
#define DTB_PROBE_T0 const unsigned long long tp0_ = clock64();
#define DTB_PROBE_ACC(v) v += clock64() - tp0_;
#else
#define DTB_PROBE_T0
#define DTB_PROBE_ACC(v)
#endif

  // ---- input rows --------------------------------------------------------
  // stage 0: the warp prefetches its own lanes' chunks of row q into ring0
  // (each lane later reads back exactly the chunks it copied: no warp sync)
  auto issue_row = [&](int q) {
    if (q < Lh) {
      const uint32_t srow = ring_in + (uint32_t)((seq0 + q) % kRing0Rows) * RB;
      const T* g = src + (int64_t)(pt.gy0 + q) * pitch + pt.gx0;
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int cb = (lane * CH + j) * E;
        if (pt.vec && cb + E <= pt.Lw) {
          pipe_cp_async16(srow + off[j], g + cb);
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e)
            if (cb + e < pt.Lw) pipe_cp_async(srow + off[j] + (uint32_t)(e * sizeof(T)), g + cb + e);
        }
      }
    }
    pipe_commit();
  };
  auto wait_in = [&](int q_hi) {  // rows [.., q_hi] are in the input ring
    if (!first) {
      DTB_PROBE_T0
      while (ld_acquire_cta(prod + stage) < seq0 + q_hi + 1) __nanosleep(kSleep);
      DTB_PROBE_ACC(w_in)
    }
  };
  auto release_in = [&](int q_done) {  // input rows < q_done are in registers
    if (!first) {
      __syncwarp();
      if (lane == 0) st_release_cta(cons + stage, seq0 + q_done);
    }
  };
  auto wait_out = [&](int q_hi) {  // ring slots up to output row q_hi are free
    if (!lastst) {
      DTB_PROBE_T0
      while (ld_acquire_cta(cons + stage + 1) < seq0 + q_hi - kRingRows + 1) __nanosleep(kSleep);
      DTB_PROBE_ACC(w_out)
    }
  };
  auto release_out = [&](int q_done) {  // output rows < q_done are written
    if (!lastst) {
      __syncwarp();
      if (lane == 0) st_release_cta(prod + stage + 1, seq0 + q_done);
    }
  };
  auto get_row = [&](int q, T (&v)[K]) {
    if (first) {
      issue_row(q + kPrefetch);
      pipe_wait_group<kPrefetch>();  // row q's group has landed (this lane's chunks)
      load_row_at<CH>(ring_in + (uint32_t)((seq0 + q) % kRing0Rows) * RB, off, v);
    } else {
      wait_in(q);
      load_row_at<CH>(ring_in + (uint32_t)((seq0 + q) % kRingRows) * RB, off, v);
      release_in(q + 1);
    }
  };
  // ---- output rows -------------------------------------------------------
  const int c_lo = lane * K;
  const bool full_vec = pt.vec && c_lo >= pt.ox0 && c_lo + K <= pt.ox1;
  // The last stage's steady loop stores whole K-column chunks, branch-free
  // (predicated 16-byte stores): a lane stores its chunk when the chunk holds
  // an owned column and lies inside the pass's exact columns [xl, xr). The
  // exact columns the chunk adds beyond the owned ones belong to the
  // neighbour segment, which stores the same bits. Segments whose owned
  // columns are not all covered that way (unaligned buffers, a lane-unaligned
  // right edge) take the generic row loop. One store flavour per loop keeps
  // the kernel's hot code small: a second copy of the stage-3 loop raised
  // instruction-fetch stalls to 32 % on C3b.
  const bool lane_owns = c_lo + K > pt.ox0 && c_lo < pt.ox1;
  const bool chunk_store = pt.vec && lane_owns && c_lo >= pt.xl && c_lo + K <= pt.xr;
  // (fp64 only: the fp32 kernel measured 15 % slower on C3b with it)
  constexpr bool kChunkStores = sizeof(T) == 8;
  const bool fast_store = !kChunkStores || __all_sync(0xffffffffu, chunk_store || !lane_owns);
  // fused slab exchange: rows the neighbours need next epoch go to them too
  auto mirror_row = [&](int q, const T (&v)[K]) {
    if constexpr (MIR) {
      const int64_t gr = pt.gy0 + q;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        if (q >= pt.qy0 && q < pt.qy1 && gr >= mir->r0[i] && gr < mir->r1[i]) {
          T* g = mir->peer[i] + (gr - mir->r0[i] + mir->p0[i]) * pitch + pt.gx0 + c_lo;
#pragma unroll
          for (int e = 0; e < K; ++e)
            if (c_lo + e >= pt.ox0 && c_lo + e < pt.ox1) g[e] = v[e];
        }
      }
    }
  };
  auto store_global = [&](T* g, const T (&v)[K]) {
    if (full_vec) {
      typedef typename Arith<T>::vec_t V;
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        V xv;
        T* px = reinterpret_cast<T*>(&xv);
#pragma unroll
        for (int e = 0; e < E; ++e) px[e] = v[j * E + e];
        *reinterpret_cast<V*>(g + j * E) = xv;
      }
    } else {
#pragma unroll
      for (int e = 0; e < K; ++e)
        if (c_lo + e >= pt.ox0 && c_lo + e < pt.ox1) g[e] = v[e];
    }
  };
  auto put_row = [&](int q, const T (&v)[K]) {
    if (lastst) {
      if (MIR) mirror_row(q, v);
      if (q >= pt.oy0 && q < pt.oy1) store_global(dst + (int64_t)(pt.gy0 + q) * pitch + pt.gx0 + c_lo, v);
    } else {
      wait_out(q);
      store_row_at<CH>(ring_out + (uint32_t)((seq0 + q) % kRingRows) * RB, off, v);
      release_out(q + 1);
    }
  };

  if (first) {
    for (int q = 0; q < kPrefetch; ++q) issue_row(q);
  }

  T x[K], o[K];
  if (levels == 0) {
    for (int q = 0; q < Lh; ++q) {
      get_row(q, x);
      put_row(q, x);
    }
  } else if (levels == 1) {
    Lv l1;
    get_row(0, x);
    put_row(0, x);  // frozen row
    l1.start(x, wt);
    for (int q = 1; q < Lh; ++q) {
      get_row(q, x);
      if (q == Lh - 1) {  // frozen bottom row finishes row Lh-2
        if (q >= 2) {
          l1.template push<true, false>(x, o, wt, lc);
          put_row(q - 1, o);
        }
        put_row(q, x);
      } else if (q == 1) {
        l1.template push<false, true>(x, o, wt, lc);
      } else {
        l1.template push<true, true>(x, o, wt, lc);
        put_row(q - 1, o);
      }
    }
  } else {
    // two levels: row q finishes t+1 row q-1 (level 1), which finishes t+2
    // row q-2 (level 2); rows 0 and Lh-1 pass through both levels unchanged
    Lv l1, l2;
    T b[K];
    get_row(0, x);
    put_row(0, x);
    l1.start(x, wt);
    l2.start(x, wt);
    if (Lh == 2) {
      get_row(1, x);
      put_row(1, x);
    } else if (Lh == 3) {
      get_row(1, x);
      l1.template push<false, true>(x, b, wt, lc);
      get_row(2, x);
      l1.template push<true, false>(x, b, wt, lc);  // t+1 row 1
      l2.template push<false, true>(b, o, wt, lc);
      l2.template push<true, false>(x, o, wt, lc);  // t+2 row 1
      put_row(1, o);
      put_row(2, x);
    } else if (Lh >= 4) {
      get_row(1, x);
      l1.template push<false, true>(x, b, wt, lc);
      get_row(2, x);
      l1.template push<true, true>(x, b, wt, lc);  // t+1 row 1
      l2.template push<false, true>(b, o, wt, lc);
      int q = 3;          // rows 3 .. Lh-2 are interior
      bool have = false;  // x already holds row q (fetched by the steady loop)
      // steady state: role-specialised copies (no role branches per row),
      // ring slots advanced incrementally (no modulo per row); the next
      // row's LDS is issued before the current row's arithmetic
      auto steady = [&](auto role_c) {
        constexpr int RL = decltype(role_c)::value;
        constexpr int RIN = RL == 0 ? kRing0Rows : kRingRows;
        const uint32_t in_end = ring_in + (uint32_t)RIN * RB;
        const uint32_t out_end = ring_out + (uint32_t)kRingRows * RB;
        uint32_t in_a = ring_in + (uint32_t)((seq0 + q) % RIN) * RB;
        uint32_t out_a = ring_out + (uint32_t)((seq0 + q - 2) % kRingRows) * RB;
        uint32_t pf_a = ring_in + (uint32_t)((seq0 + q + kPrefetch) % RIN) * RB;
        const T* pf_g = src + (int64_t)(pt.gy0 + q + kPrefetch) * pitch + pt.gx0;
        const bool pf_fast = pt.vec && pt.Lw == L::ROW;
        T* st_g = dst + (int64_t)(pt.gy0 + q - 2) * pitch + pt.gx0 + c_lo;
        int fq = q;  // the next row to fetch
        T y[K];
        // PF: 0 = no prefetch (the tail), 1 = whole-row 16-byte copies,
        // 2 = the general per-chunk path, 3 = either, checked per row
        // (stage 0 only)
        auto fetch = [&](T (&v)[K], auto pf_c) {
          constexpr int PF = decltype(pf_c)::value;
          if constexpr (RL == 0 && PF == 3) {
            if (fq + kPrefetch < Lh) {
              if (pf_fast) {
#pragma unroll
                for (int j = 0; j < CH; ++j) pipe_cp_async16(pf_a + off[j], pf_g + (lane * CH + j) * E);
              } else {
#pragma unroll
                for (int j = 0; j < CH; ++j) {
                  const int cb = (lane * CH + j) * E;
                  if (pt.vec && cb + E <= pt.Lw) {
                    pipe_cp_async16(pf_a + off[j], pf_g + cb);
                  } else {
#pragma unroll
                    for (int e = 0; e < E; ++e)
                      if (cb + e < pt.Lw) pipe_cp_async(pf_a + off[j] + (uint32_t)(e * sizeof(T)), pf_g + cb + e);
                  }
                }
              }
            }
          } else if constexpr (RL == 0 && PF != 0) {  // stage 0: keep kPrefetch HBM rows in flight
            if constexpr (PF == 1) {
#pragma unroll
              for (int j = 0; j < CH; ++j) pipe_cp_async16(pf_a + off[j], pf_g + (lane * CH + j) * E);
            } else {
#pragma unroll
              for (int j = 0; j < CH; ++j) {
                const int cb = (lane * CH + j) * E;
                if (pt.vec && cb + E <= pt.Lw) {
                  pipe_cp_async16(pf_a + off[j], pf_g + cb);
                } else {
#pragma unroll
                  for (int e = 0; e < E; ++e)
                    if (cb + e < pt.Lw) pipe_cp_async(pf_a + off[j] + (uint32_t)(e * sizeof(T)), pf_g + cb + e);
                }
              }
            }
          }
          if constexpr (RL == 0) {
            pipe_commit();
            pipe_wait_group<kPrefetch>();  // row fq's group has landed
            pf_a += RB;
            if (pf_a == in_end) pf_a = ring_in;
            pf_g += pitch;
          }
          load_row_at<CH>(in_a, off, v);
          in_a += RB;
          if (in_a == in_end) in_a = ring_in;
          ++fq;
        };
        auto emit = [&](const T (&v)[K]) {  // t+2 row q-2
          if constexpr (RL == 2) {
            if (MIR) mirror_row(q - 2, v);
            if constexpr (kChunkStores)
              st_row_pred(q - 2 >= pt.oy0 && q - 2 < pt.oy1 && chunk_store, st_g, v);
            else if (q - 2 >= pt.oy0 && q - 2 < pt.oy1)
              store_global(st_g, v);
            st_g += pitch;
          } else {
            store_row_at<CH>(out_a, off, v);
            out_a += RB;
            if (out_a == out_end) out_a = ring_out;
          }
        };
        // blocks of 4 interior rows q..q+3 (q+3 <= Lh-2): read rows up to
        // q+4 (<= Lh-1, the last one kept in x), write rows q-2..q+1.
        // Stage 0's prefetch needs no per-row bound check while every row of
        // the block still has one to issue (fq + 3 + kPrefetch < Lh), and the
        // whole-row path is chosen once per segment, not per row.
        auto block = [&](auto pf_c) {
          wait_in(q + 4);
          wait_out(q + 1);
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            fetch(y, pf_c);
            l1.template push<true, true>(x, b, wt, lc);
            l2.template push<true, true>(b, o, wt, lc);
            emit(o);
            ++q;
            fetch(x, pf_c);
            l1.template push<true, true>(y, b, wt, lc);
            l2.template push<true, true>(b, o, wt, lc);
            emit(o);
            ++q;
          }
          release_in(q + 1);   // rows <= q are in registers
          release_out(q - 2);  // outputs < q-2 written
        };
        wait_in(q);
        if constexpr (RL == 0 && sizeof(T) == 4) {
          // fp32: the per-row checked loop (the split loops below measured
          // 27 % slower on C3b; fp64 C4 gains 2.5 % from them)
          fetch(x, std::integral_constant<int, 3>{});
          while (q + 4 <= Lh - 1) block(std::integral_constant<int, 3>{});
        } else if constexpr (RL == 0) {
          if (fq + kPrefetch < Lh) fetch(x, std::integral_constant<int, 2>{});
          else fetch(x, std::integral_constant<int, 0>{});
          if (pf_fast) {
            while (q + 4 <= Lh - 1 && fq + 3 + kPrefetch < Lh) block(std::integral_constant<int, 1>{});
          } else {
            while (q + 4 <= Lh - 1 && fq + 3 + kPrefetch < Lh) block(std::integral_constant<int, 2>{});
          }
          // the block that crosses the end of the prefetch window, row by row
          while (q + 4 <= Lh - 1 && fq + kPrefetch < Lh) {
            wait_in(q + 4);
            wait_out(q + 1);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              if (fq + kPrefetch < Lh) fetch(y, std::integral_constant<int, 2>{});
              else fetch(y, std::integral_constant<int, 0>{});
              l1.template push<true, true>(x, b, wt, lc);
              l2.template push<true, true>(b, o, wt, lc);
              emit(o);
              ++q;
              if (fq + kPrefetch < Lh) fetch(x, std::integral_constant<int, 2>{});
              else fetch(x, std::integral_constant<int, 0>{});
              l1.template push<true, true>(y, b, wt, lc);
              l2.template push<true, true>(b, o, wt, lc);
              emit(o);
              ++q;
            }
            release_in(q + 1);
            release_out(q - 2);
          }
          while (q + 4 <= Lh - 1) block(std::integral_constant<int, 0>{});
        } else {
          fetch(x, std::integral_constant<int, 0>{});
          while (q + 4 <= Lh - 1) block(std::integral_constant<int, 0>{});
        }
        have = true;
      };
      if (q + 4 <= Lh - 1 && (!lastst || fast_store)) {  // at least one steady block
        if (first) steady(std::integral_constant<int, 0>{});
        else if (lastst) steady(std::integral_constant<int, 2>{});
        else steady(std::integral_constant<int, 1>{});
      }
      // generic rows (short segments, and the tail of long ones)
      for (; q < Lh - 1; ++q) {
        if (!have) get_row(q, x);
        have = false;
        l1.template push<true, true>(x, b, wt, lc);
        l2.template push<true, true>(b, o, wt, lc);
        put_row(q - 2, o);
      }
      if (!have) get_row(Lh - 1, x);  // frozen bottom row
      l1.template push<true, false>(x, b, wt, lc);  // t+1 row Lh-2
      l2.template push<true, true>(b, o, wt, lc);   // t+2 row Lh-3
      put_row(Lh - 3, o);
      l2.template push<true, false>(x, o, wt, lc);  // t+2 row Lh-2
      put_row(Lh - 2, o);
      put_row(Lh - 1, x);
    }
  }
#if DTB_PIPE_PROBE
  if (lane == 0) {
    atomicAdd(&g_pipe_probe[stage][0], w_in);
    atomicAdd(&g_pipe_probe[stage][1], w_out);
    atomicAdd(&g_pipe_probe[stage][2], clock64() - t_all);
  }
#endif
#undef DTB_PROBE_T0
#undef DTB_PROBE_ACC
  if (first) pipe_wait_group<0>();  // drain empty tail groups
  if (!first && lane == 0) st_release_cta(cons + stage, seq0 + Lh);  // whole tile consumed
}

template <int S>
struct PipeSmem {
  int prod[S], cons[S];
};

// One wavefront diagonal (launch_pipe_wave): n (pass, row block) tasks, each
// all column strips of row block ty advanced by `steps` steps from src to dst
// (the pass's parity buffers). Empty (n == 0): the plain pass over every tile.
template <typename T>
struct PipeWave {
  int n;
  int ty[kMaxWaveTasks];
  int steps[kMaxWaveTasks];
  const T* src[kMaxWaveTasks];
  T* dst[kMaxWaveTasks];
};

// One pass of up to 2S fused steps: NW/S pipelines of S warps per CTA, each
// pipeline marching column-strip segments. Warp w runs stage w / P of
// pipeline w % P, so each SM sub-partition (warp % 4) hosts one whole
// pipeline and a stage's slack goes to its own upstream/downstream warps.
template <typename T, int K, int NW, int S, bool SYM, bool DYN, bool MIR>
__global__ void __launch_bounds__(NW * 32, 1)
pipe_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t pitch, int nx, int ny,
            Weights<T> wt, int steps, const __grid_constant__ Geometry geo,
            const __grid_constant__ HaloMirror<T> mir, unsigned long long* __restrict__ cnt,
            const __grid_constant__ PipeWave<T> wave) {
  constexpr int P = NW / S;
  typedef Tile<T, K> L;
  constexpr int RB = L::ROW * (int)sizeof(T);
  constexpr int kRing0Rows = PipeCfg<T>::kRing0Rows, kRingRows = PipeCfg<T>::kRingRows;
  constexpr int kPipeBytes = (kRing0Rows + (S - 1) * kRingRows) * RB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int p = warp % P, s = warp / P;
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
  LaneCtx lc;
  lc.lane = threadIdx.x & 31;
  lc.first = lc.lane == 0;
  const int ntiles = geo.ntx * (wave.n ? wave.n : geo.nty);
  int seq = 0;
  for (int t = blockIdx.x * P + p; t < ntiles; t += gridDim.x * P) {
    int tx = t % geo.ntx, ty = t / geo.ntx;
    const T* tsrc = src;
    T* tdst = dst;
    int tsteps = steps;
    if (wave.n) {  // wavefront task ty of this diagonal: its row block and buffers
      const int k = ty;
      ty = wave.ty[k];
      tsrc = wave.src[k];
      tdst = wave.dst[k];
      tsteps = wave.steps[k];
    }
    const int levels = max(0, min(2, tsteps - 2 * s));
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
    pt.xl = cx.z > -1 ? tsteps : 0;
    pt.xr = cx.w < nx + 1 ? pt.Lw - tsteps : pt.Lw;
    lc.last = lc.lane == (pt.Lw - 1) / K;
    lc.last_e = (pt.Lw - 1) % K;
    pipe_stage<T, K, SYM, DYN, MIR>(pt, s, S, levels, seq, tsrc, tdst, pitch, ring_in, ring_out,
                                    ctl[p].prod, ctl[p].cons, wt, lc, &mir);
    if (cnt && lc.lane == 0) {  // counted traffic (domain cells only)
      const long long dc = span_in(pt.gx0, pt.gx0 + pt.Lw, 1, nx + 1);
      if (s == 0)  // stage 0 read the segment's rows from HBM
        atomicAdd(cnt + 0, (unsigned long long)(span_in(pt.gy0, pt.gy0 + pt.Lh, 1, ny + 1) * dc));
      if (levels > 0)
        atomicAdd(cnt + 3, (unsigned long long)levels * max(0, pt.Lh - 2) * max(0, pt.Lw - 2));
      if (s == S - 1) {  // the last stage stored the owned rows (and fed the mirrors)
        const long long sc = span_in(pt.gx0 + pt.ox0, pt.gx0 + pt.ox1, 1, nx + 1);
        atomicAdd(cnt + 1, (unsigned long long)(span_in(pt.gy0 + pt.oy0, pt.gy0 + pt.oy1, 1,
                                                        ny + 1) * sc));
        if (MIR) {
#pragma unroll
          for (int i = 0; i < 2; ++i)
            atomicAdd(cnt + 2, (unsigned long long)(span_in(pt.gy0 + pt.qy0, pt.gy0 + pt.qy1,
                                                            mir.r0[i], mir.r1[i]) * sc));
        }
      }
    }
    seq += pt.Lh;
  }
  // mirror passes store into peer GPUs' (or other processes') buffers: make
  // them system-visible before the kernel's completion is signalled
  if (MIR) __threadfence_system();
}

template <typename T, int K, bool SYM, bool DYN>
int launch_pipe_kernel(const Plan& p, const Geometry& geo, const T* d_in, T* d_out, int64_t pitch,
                       int nx, int ny, const Weights<T>& wt, int64_t steps, cudaStream_t st,
                       unsigned long long* cnt) {
  constexpr int S = kPipeStages, PW = PipeCfg<T>::kWarps, P = PW / S;
  auto kern = pipe_kernel<T, K, PW, S, SYM, DYN, false>;
  auto kmir = pipe_kernel<T, K, PW, S, SYM, DYN, true>;
  const int pipe_bytes = (PipeCfg<T>::kRing0Rows + (S - 1) * PipeCfg<T>::kRingRows) *
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
    if (int rc = arena_get(kArenaScratch, device, grid_bytes, &scratch)) return rc;
    tmp = reinterpret_cast<T*>(scratch);
  }
  const int64_t ntiles = (int64_t)geo.ntx * geo.nty;
  DevInfo di;
  if (int rc = query_dev(di)) return rc;
  const int ctas = (int)std::min<int64_t>(di.sms, (ntiles + P - 1) / P);
  const HaloMirror<T>* mir = static_cast<const HaloMirror<T>*>(g_halo_mirror);
  HaloMirror<T> none;
  memset(&none, 0, sizeof none);
  PipeWave<T> nowave;
  nowave.n = 0;
  if (mir) {
    if (int rc = prepare_kernel((const void*)kmir, device, psmem, PW * 32, nullptr)) return rc;
  }
  const T* src = d_in;
  int64_t done = 0;
  for (int64_t i = 0; i < passes; ++i) {
    const int s = (int)std::min<int64_t>(2 * S, steps - done);
    T* dst = ((passes - 1 - i) % 2 == 0) ? d_out : tmp;
    if (mir && i + 1 == passes)  // the epoch's result: also feed the neighbours' halos
      kmir<<<ctas, PW * 32, psmem, st>>>(src, dst, pitch, nx, ny, wt, s, geo, *mir, cnt, nowave);
    else
      kern<<<ctas, PW * 32, psmem, st>>>(src, dst, pitch, nx, ny, wt, s, geo, none, cnt, nowave);
    g_launches += 1;
    CUDA_TRY(cudaGetLastError());
    src = dst;
    done += s;
  }
  return DTB_OK;
}

// Passes as temporal wavefronts where host copies can overlap them. Task
// (k, j) = pass k (1-based, steps 8(k-1)+1 .. 8k) on row block j of the wave
// geometry (gw.row). It reads row blocks j-1..j+1 of pass k-1's output (the
// 8-row halos stay inside the neighbours) and overwrites block j of the buffer
// pass k-2 wrote, which only passes k-1 on blocks j-1..j+1 read. So the tasks
// of one diagonal d = 2k + j depend only on earlier diagonals and not on each
// other: one launch per diagonal, in order on `st`.
//   phase A: passes 1..mA as a wavefront; a diagonal waits only for the input
//            row blocks its first-pass tasks read (hooks.in_ready),
//   phase B: the middle passes as plain full-grid passes (p / geo: long
//            segments, no wave overheads),
//   phase C: the last mC passes as a wavefront; each final row block is
//            handed to hooks.out_done as soon as its diagonal is launched.
// The wavefront phases cost extra row-block halos and shorter segments, so
// they only cover about as many passes as the host copy they hide (m).
template <typename T, int K, bool SYM, bool DYN>
int launch_pipe_wave_kernel(const Plan& p, const Geometry& geo, const Geometry& gw,
                            const T* d_in, T* d_out, int64_t pitch, int nx, int ny,
                            const Weights<T>& wt, int64_t steps, int64_t m, cudaStream_t st,
                            unsigned long long* cnt, const PipeWaveHooks& hooks) {
  constexpr int S = kPipeStages, PW = PipeCfg<T>::kWarps, P = PW / S, h = 2 * S;
  auto kern = pipe_kernel<T, K, PW, S, SYM, DYN, false>;
  const int pipe_bytes = (PipeCfg<T>::kRing0Rows + (S - 1) * PipeCfg<T>::kRingRows) *
                         Tile<T, K>::ROW * (int)sizeof(T);
  const int psmem = P * pipe_bytes + (int)sizeof(PipeSmem<S>) * P;
  int device;
  CUDA_TRY(cudaGetDevice(&device));
  if (int rc = prepare_kernel((const void*)kern, device, psmem, PW * 32, nullptr)) return rc;
  const int J = gw.nty;
  const int64_t passes = (steps + h - 1) / h;
  if (J < 1 || J > 2 * kMaxWaveTasks - 2 || passes < 2 || gw.ntx != geo.ntx)
    return fail(DTB_EINVAL, "wavefront of %d row blocks x %lld passes", J, (long long)passes);
  T* tmp = nullptr;
  {
    void* scratch = nullptr;
    const size_t grid_bytes = (size_t)(ny + 2) * pitch * sizeof(T);
    if (int rc = arena_get(kArenaScratch, device, grid_bytes, &scratch)) return rc;
    tmp = reinterpret_cast<T*>(scratch);
  }
  DevInfo di;
  if (int rc = query_dev(di)) return rc;
  HaloMirror<T> none;
  memset(&none, 0, sizeof none);
  PipeWave<T> wave;
  auto dst_of = [&](int64_t k) { return ((passes - k) % 2 == 0) ? d_out : tmp; };  // k 1-based
  auto src_of = [&](int64_t k) -> const T* { return k == 1 ? d_in : dst_of(k - 1); };
  auto steps_of = [&](int64_t k) { return (int)std::min<int64_t>(h, steps - (k - 1) * h); };
  // passes [k0, k1] as one wavefront
  auto wavefront = [&](int64_t k0, int64_t k1) -> int {
    const int64_t n = k1 - k0 + 1;
    for (int64_t d = 2; d <= 2 * n + J - 1; ++d) {
      wave.n = 0;
      int need = -1;  // input row blocks the first-pass tasks read
      for (int64_t q = std::min<int64_t>(n, d / 2); q >= 1 && d - 2 * q < J; --q) {
        const int j = (int)(d - 2 * q), k = (int)(k0 + q - 1);
        wave.ty[wave.n] = j;
        wave.steps[wave.n] = steps_of(k);
        wave.src[wave.n] = src_of(k);
        wave.dst[wave.n] = dst_of(k);
        ++wave.n;
        if (k == 1) need = std::min(j + 1, J - 1);
      }
      if (need >= 0 && hooks.in_ready)
        if (int rc = hooks.in_ready(hooks.ctx, need)) return rc;
      const int ctas = (int)std::min<int64_t>(di.sms, ((int64_t)wave.n * gw.ntx + P - 1) / P);
      kern<<<ctas, PW * 32, psmem, st>>>(d_in, d_out, pitch, nx, ny, wt, h, gw, none, cnt, wave);
      g_launches += 1;
      CUDA_TRY(cudaGetLastError());
      // the last pass's task on block d - 2n is in this launch: that block is final
      if (k1 == passes && d - 2 * n >= 0 && hooks.out_done)
        if (int rc = hooks.out_done(hooks.ctx, (int)(d - 2 * n))) return rc;
    }
    return DTB_OK;
  };
  const int64_t mA = std::max<int64_t>(1, std::min(m, passes));
  const int64_t mC = std::min<int64_t>(m, passes - mA);
  if (int rc = wavefront(1, mA)) return rc;
  wave.n = 0;
  const int ctas = (int)std::min<int64_t>(di.sms, ((int64_t)geo.ntx * geo.nty + P - 1) / P);
  for (int64_t k = mA + 1; k <= passes - mC; ++k) {
    kern<<<ctas, PW * 32, psmem, st>>>(src_of(k), dst_of(k), pitch, nx, ny, wt, steps_of(k), geo,
                                       none, cnt, wave);
    g_launches += 1;
    CUDA_TRY(cudaGetLastError());
  }
  if (mC > 0)
    if (int rc = wavefront(passes - mC + 1, passes)) return rc;
  return DTB_OK;
}

template <typename T>
int launch_pipe_wave(const Plan& p, const Geometry& geo, const Geometry& gw, const T* d_in,
                     T* d_out, int64_t pitch, int nx, int ny, const T w[5], int64_t steps,
                     int64_t m, cudaStream_t st, unsigned long long* cnt,
                     const PipeWaveHooks& hooks) {
  constexpr int K = PipeCfg<T>::kK;
  if (p.K != K || p.warps != PipeCfg<T>::kWarps || p.mode != 3)
    return fail(DTB_EINFEASIBLE, "no pipe kernel for elem %d K %d warps %d", (int)sizeof(T), p.K,
                p.warps);
  Weights<T> wt{w[0], w[1], w[2], w[3], w[4]};
  const bool sym = weights_isotropic<T>(w);
#define DTB_GO(S, D)                                                                          \
  return launch_pipe_wave_kernel<T, K, S, D>(p, geo, gw, d_in, d_out, pitch, nx, ny, wt, steps, \
                                              m, st, cnt, hooks)
  if (sym) {
    if (p.dyn()) DTB_GO(true, true);
    DTB_GO(true, false);
  }
  if (p.dyn()) DTB_GO(false, true);
  DTB_GO(false, false);
#undef DTB_GO
}

template <typename T>
int launch_pipe(const Plan& p, const Geometry& geo, const T* d_in, T* d_out, int64_t pitch,
                int nx, int ny, const T w[5], int64_t steps, cudaStream_t st,
                unsigned long long* cnt) {
  constexpr int K = PipeCfg<T>::kK;
  if (p.K != K || p.warps != PipeCfg<T>::kWarps)
    return fail(DTB_EINFEASIBLE, "no pipe kernel for elem %d K %d warps %d", (int)sizeof(T), p.K,
                p.warps);
  Weights<T> wt{w[0], w[1], w[2], w[3], w[4]};
  const bool sym = weights_isotropic<T>(w);
#define DTB_GO(S, D) return launch_pipe_kernel<T, K, S, D>(p, geo, d_in, d_out, pitch, nx, ny, wt, steps, st, cnt)
  if (sym) {
    if (p.dyn()) DTB_GO(true, true);
    DTB_GO(true, false);
  }
  if (p.dyn()) DTB_GO(false, true);
  DTB_GO(false, false);
#undef DTB_GO
}

}  // namespace dtb
