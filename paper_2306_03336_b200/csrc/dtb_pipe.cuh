// dtb_pipe.cuh — the pipelined (2.5-D) streaming kernel.
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
// Compared with the tile sweep (dtb_core.cuh) there are no band seams, no
// CTA-wide barriers and no pre-read halo registers; y-redundancy exists only
// at segment ends (segments are hundreds to thousands of rows) and the HBM
// traffic of a pass is one read + one write of every owned cell, overlapped
// with the FP work by the ring prefetch. Each warp spans the strip width
// (32*K columns, lane-owned K-column chunks, shuffles for W/E) exactly as in
// the tile sweep; every update is the same FMA-free W,E,S,C,N expression
// (kernel.py:137-139), so results stay bitwise equal to jacobi_reference.
//
// Synchronisation inside a pipeline is by monotonic row counters in shared
// memory (st.release.cta / ld.acquire.cta): prod[s] = rows written into ring
// s, cons[s] = rows ring s's reader no longer needs.
#pragma once
#include "dtb_core.cuh"
#include <type_traits>

namespace dtb {

__device__ __forceinline__ void pipe_cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void pipe_cp_async(uint32_t dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void pipe_cp_async(uint32_t dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
template <int N>
__device__ __forceinline__ void pipe_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void pipe_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

// Ring geometry (rows of 32*K elements, the tile row layout incl. swizzle),
// per CTA width: 8 warps = 2 pipelines with deep rings, 16 warps = 4
// pipelines with shallower rings (the smem budget). Block-level flow control
// needs kRingRows >= 12 to stay deadlock-free (see pipe_stage).
// fp64 rows need a deeper HBM prefetch than fp32 rows (same 1 KB per row, half
// the cells, so half the compute per row to hide a row's latency behind)
#ifndef DTB_PIPE_R0
#define DTB_PIPE_R0 16
#endif
#ifndef DTB_PIPE_PF
#define DTB_PIPE_PF 10
#endif
#ifndef DTB_PIPE_RING
#define DTB_PIPE_RING 12
#endif
template <int NW, typename T = double>
struct PipeCfg {
  static constexpr bool kDeep = NW >= 16 && sizeof(T) == 8;
  static constexpr int kRing0Rows = NW >= 16 ? (kDeep ? DTB_PIPE_R0 : 12) : 16;  // stage 0's HBM prefetch ring
  static constexpr int kRingRows = NW >= 16 ? (kDeep ? DTB_PIPE_RING : 12) : 16;  // ring between stages
  static constexpr int kPrefetch = NW >= 16 ? (kDeep ? DTB_PIPE_PF : 6) : 8;  // HBM rows in flight
};

// Fused slab halo exchange (n_gpus > 1 through the C ABI): the last stage
// also stores padded rows [r0[i], r1[i]) of its output into a neighbour
// slab's next input at rows p0[i].. (a peer GPU's buffer over NVLink, or the
// same device when slabs share one), and stores its own rows only inside
// [sw0, sw1) so it never touches the halo rows the neighbours write.
template <typename T>
struct HaloMirror {
  T* peer[2];
  int64_t r0[2], r1[2], p0[2];
  int64_t sw0, sw1;
};

struct PipeTile {
  int Lw, Lh;        // load region (tile-local rows/cols)
  int gx0, gy0;      // padded global coords of tile (0,0)
  int ox0, ox1;      // store columns (owned, + ghost at domain edges), tile-local
  int oy0, oy1;      // store rows, tile-local
  int qy0, qy1;      // owned rows, tile-local (oy before a HaloMirror store window)
  bool vec;          // global side 16-byte aligned per chunk
};

// One pipeline stage warp advancing one tile by `levels` (0, 1 or 2) steps.
// seq0: the pipeline-wide row sequence number of this tile's row 0 (ring
// slot = seq % ring rows). `src` is read only by stage 0; `dst` written only
// by the last stage.
// ROLE: 0 first stage (HBM prefetch in), 1 middle, 2 last stage (STG out);
// resolved at compile time so the steady loop carries no role branches.
#ifndef DTB_PIPE_NOINLINE
#define DTB_PIPE_NOINLINE 0
#endif
#ifndef DTB_PIPE_PROBE
#define DTB_PIPE_PROBE 0  // per-stage wait-cycle counters (dtb_debug_pipe_probe)
#endif
#if DTB_PIPE_PROBE
__device__ unsigned long long g_pipe_probe[8][3];
#endif
#if DTB_PIPE_NOINLINE
#define DTB_PIPE_INL __noinline__
#else
#define DTB_PIPE_INL __forceinline__
#endif
template <typename T, int K, int NW, bool DYN, int ROLE, bool MIR = false>
__device__ DTB_PIPE_INL void pipe_stage_role(const PipeTile& pt, int stage, int levels,
                                                int seq0, const T* __restrict__ src,
                                                T* __restrict__ dst, int64_t pitch,
                                                uint32_t ring_in, uint32_t ring_out, int* prod,
                                                int* cons, const Weights<T>& wt,
                                                const LaneCtx& lc, int nstages_,
                                                const HaloMirror<T>* mir = nullptr) {
  typedef Tile<T, K> L;
  constexpr int E = L::EPC, CH = L::CH;
  constexpr uint32_t RB = (uint32_t)(L::ROW * sizeof(T));  // bytes per ring row
  const int lane = lc.lane;
  const int Lh = pt.Lh;
  uint32_t off[CH];
#pragma unroll
  for (int j = 0; j < CH; ++j) off[j] = (uint32_t)(L::swz(lane * CH + j) * 16);
#ifndef DTB_PIPE_ROLES
#define DTB_PIPE_ROLES 0  // 1: stage role as a template parameter (spills at 128 registers)
#endif
  const bool first = DTB_PIPE_ROLES ? ROLE == 0 : stage == 0;
  const bool lastst = DTB_PIPE_ROLES ? ROLE == 2 : stage == nstages_ - 1;
  constexpr int kRing0Rows = PipeCfg<NW, T>::kRing0Rows, kRingRows = PipeCfg<NW, T>::kRingRows,
                kPrefetch = PipeCfg<NW, T>::kPrefetch;

  // ---- input rows --------------------------------------------------------
  // stage 0: the warp prefetches its own lanes' chunks of row q into ring0
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
  // block-level flow control (steady loop): wait until rows [.., q_hi] are in
  // the input ring / ring slots up to output row q_hi are free
#ifndef DTB_PIPE_ROW2
// steady rows: 1 stage-major pair update, 0 two row updates (fp64 faster
// with two, fp32 with the pair: B200 A/B, round 1)
#define DTB_PIPE_ROW2 (sizeof(T) == 4)
#endif
#ifndef DTB_PIPE_SPEC
#define DTB_PIPE_SPEC 1  // role-specialised steady loops, incremental ring slots
#endif
#ifndef DTB_PIPE_SLEEP
#define DTB_PIPE_SLEEP 400  // ns between ring-counter polls (fp32 +2.5 %, fp64 flat vs 20)
#endif
#ifndef DTB_PIPE_POLL
#define DTB_PIPE_POLL 1  // 1: every lane polls (warp-uniform loop); 0: lane 0 polls + syncwarp
#endif
#if DTB_PIPE_PROBE
  unsigned long long w_in = 0, w_out = 0, t_all = clock64();
#define DTB_PROBE_T0 const unsigned long long tp0_ = clock64();
#define DTB_PROBE_ACC(v) v += clock64() - tp0_;
#else
#define DTB_PROBE_T0
#define DTB_PROBE_ACC(v)
#endif
  auto wait_in = [&](int q_hi) {
    if (!first) {
      DTB_PROBE_T0
      if (DTB_PIPE_POLL) {
        while (ld_acquire_cta(prod + stage) < seq0 + q_hi + 1) __nanosleep(DTB_PIPE_SLEEP);
      } else {
        if (lane == 0)
          while (ld_acquire_cta(prod + stage) < seq0 + q_hi + 1) __nanosleep(DTB_PIPE_SLEEP);
        __syncwarp();
      }
      DTB_PROBE_ACC(w_in)
    }
  };
  auto release_in = [&](int q_done) {  // input rows < q_done fully read
    if (!first) {
      __syncwarp();
      if (lane == 0) st_release_cta(cons + stage, seq0 + q_done);
    }
  };
  auto wait_out = [&](int q_hi) {
    if (!lastst) {
      DTB_PROBE_T0
      if (DTB_PIPE_POLL) {
        while (ld_acquire_cta(cons + stage + 1) < seq0 + q_hi - kRingRows + 1) __nanosleep(DTB_PIPE_SLEEP);
      } else {
        if (lane == 0)
          while (ld_acquire_cta(cons + stage + 1) < seq0 + q_hi - kRingRows + 1) __nanosleep(DTB_PIPE_SLEEP);
        __syncwarp();
      }
      DTB_PROBE_ACC(w_out)
    }
  };
  auto release_out = [&](int q_done) {  // output rows < q_done written
    if (!lastst) {
      __syncwarp();
      if (lane == 0) st_release_cta(prod + stage + 1, seq0 + q_done);
    }
  };
  auto get_row_nosync = [&](int q, T (&v)[K]) {
    if (first) {
      issue_row(q + kPrefetch);
      pipe_wait_group<kPrefetch>();  // row q's group has landed (this lane's chunks)
      load_row_at<CH>(ring_in + (uint32_t)((seq0 + q) % kRing0Rows) * RB, off, v);
    } else {
      load_row_at<CH>(ring_in + (uint32_t)((seq0 + q) % kRingRows) * RB, off, v);
    }
  };
  auto get_row = [&](int q, T (&v)[K]) {
    wait_in(q);
    get_row_nosync(q, v);
    // rows up to q-2 are in registers and no longer read from the ring
    if (q >= 2) release_in(q - 1);
  };
  // ---- output rows -------------------------------------------------------
  const int c_lo = lane * K;
  const bool full_vec = pt.vec && c_lo >= pt.ox0 && c_lo + K <= pt.ox1;
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
  auto put_row_nosync = [&](int q, const T (&v)[K]) {
    if (lastst) {
      if (MIR) mirror_row(q, v);
      if (q >= pt.oy0 && q < pt.oy1) {
        T* g = dst + (int64_t)(pt.gy0 + q) * pitch + pt.gx0 + c_lo;
        if (full_vec) {
          typedef typename Arith<T>::vec_t V;
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            V x;
            T* px = reinterpret_cast<T*>(&x);
#pragma unroll
            for (int e = 0; e < E; ++e) px[e] = v[j * E + e];
            *reinterpret_cast<V*>(g + j * E) = x;
          }
        } else {
#pragma unroll
          for (int e = 0; e < K; ++e)
            if (c_lo + e >= pt.ox0 && c_lo + e < pt.ox1) g[e] = v[e];
        }
      }
    } else {
      store_row_at<CH>(ring_out + (uint32_t)((seq0 + q) % kRingRows) * RB, off, v);
    }
  };
  auto put_row = [&](int q, const T (&v)[K]) {
    wait_out(q);
    put_row_nosync(q, v);
    release_out(q + 1);
  };

  if (first) {
    for (int q = 0; q < kPrefetch; ++q) issue_row(q);
  }

  if (levels == 0) {
    for (int q = 0; q < Lh; ++q) {
      T v[K];
      get_row(q, v);
      put_row(q, v);
    }
  } else if (levels == 1) {
    T a0[K], a1[K], a2[K], o[K];
    get_row(0, a1);
    put_row(0, a1);  // frozen row
    if (Lh > 1) get_row(1, a2);
    for (int q = 1; q + 1 < Lh; ++q) {
      copy_row<T, K>(a1, a0);
      copy_row<T, K>(a2, a1);
      get_row(q + 1, a2);
      row_update<T, K, DYN>(a0, a1, a2, o, wt, lc);
      put_row(q, o);
    }
    if (Lh > 1) put_row(Lh - 1, a2);  // frozen row
  } else {
    // two levels, skewed: iteration r loads t(r+2), computes b(r) = L1(t) and
    // out(r-2) = L2(b); t(q) in T[q%4], b(q) in B[q%4] (static after unroll)
    T t0[K], t1[K], t2[K], t3[K], b0[K], b1[K], b2[K], b3[K], o[K];
    get_row(0, t0);
    if (Lh > 1) get_row(1, t1);
#define DTB_PIPE_ITER(TM1, TC, TP1, TP2, BR, BM1, BM2, BM3)                       \
  {                                                                               \
    if (r + 2 < Lh) get_row(r + 2, TP2);                                          \
    if (r < Lh) {                                                                 \
      if (r == 0 || r == Lh - 1) copy_row<T, K>(TC, BR);                          \
      else row_update<T, K, DYN>(TM1, TC, TP1, BR, wt, lc);                       \
    }                                                                             \
    if (r >= 2 && r - 2 < Lh) {                                                   \
      if (r - 2 == 0 || r - 2 == Lh - 1) put_row(r - 2, BM2);                     \
      else {                                                                      \
        row_update<T, K, DYN>(BM3, BM2, BM1, o, wt, lc);                          \
        put_row(r - 2, o);                                                        \
      }                                                                           \
    }                                                                             \
    ++r;                                                                          \
  }
#define DTB_PIPE_STEADY(TM1, TC, TP1, TP2, BR, BM1, BM2, BM3)                     \
  {                                                                               \
    get_row_nosync(r + 2, TP2);                                                   \
    if (DTB_PIPE_ROW2) {                                                          \
      row_update2<T, K, DYN>(TM1, TC, TP1, BR, BM3, BM2, BM1, o, wt, lc);         \
    } else {                                                                      \
      row_update<T, K, DYN>(TM1, TC, TP1, BR, wt, lc);                            \
      row_update<T, K, DYN>(BM3, BM2, BM1, o, wt, lc);                            \
    }                                                                             \
    put_row_nosync(r - 2, o);                                                     \
    ++r;                                                                          \
  }
    // slots at iteration r (mod 4): r%4==0: (t3,t0,t1,t2, b0,b3,b2,b1)
    //   r%4==1: (t0,t1,t2,t3, b1,b0,b3,b2)  r%4==2: (t1,t2,t3,t0, b2,b1,b0,b3)
    //   r%4==3: (t2,t3,t0,t1, b3,b2,b1,b0)
    int r = 0;
    // prologue r = 0..3 (frozen row 0, first L2 rows)
    DTB_PIPE_ITER(t3, t0, t1, t2, b0, b3, b2, b1)
    DTB_PIPE_ITER(t0, t1, t2, t3, b1, b0, b3, b2)
    DTB_PIPE_ITER(t1, t2, t3, t0, b2, b1, b0, b3)
    DTB_PIPE_ITER(t2, t3, t0, t1, b3, b2, b1, b0)
    // steady: r .. r+3 all interior (r-2 >= 1, r+3+2 < Lh, r+3 < Lh-1)
#if DTB_PIPE_SPEC
    // role-specialised copies of the steady loop (no role branches per row)
    // with ring slots advanced incrementally (no modulo per row)
    auto steady = [&](auto role_c) {
      constexpr int RL = decltype(role_c)::value;
      constexpr int RIN = RL == 0 ? kRing0Rows : kRingRows;
      const uint32_t in_end = ring_in + (uint32_t)RIN * RB;
      const uint32_t out_end = ring_out + (uint32_t)kRingRows * RB;
      uint32_t in_a = ring_in + (uint32_t)((seq0 + r + 2) % RIN) * RB;
      uint32_t out_a = ring_out + (uint32_t)((seq0 + r - 2) % kRingRows) * RB;
      uint32_t pf_a = ring_in + (uint32_t)((seq0 + r + 2 + kPrefetch) % RIN) * RB;
      const T* pf_g = src + (int64_t)(pt.gy0 + r + 2 + kPrefetch) * pitch + pt.gx0;
      const bool pf_fast = sizeof(T) == 8 && pt.vec && pt.Lw == L::ROW;  // fp32: slower (B200 A/B)
      T* st_g = dst + (int64_t)(pt.gy0 + r - 2) * pitch + pt.gx0 + c_lo;
#define DTB_PIPE_SPEC_ROW(TM1, TC, TP1, TP2, BR, BM1, BM2, BM3)                   \
  {                                                                               \
    if constexpr (RL == 0) {                                                      \
      if (r + 2 + kPrefetch < Lh) {                                               \
        if (pf_fast) {  /* full-width aligned strip: CH chunk copies, no checks */\
          _Pragma("unroll") for (int j = 0; j < CH; ++j)                          \
              pipe_cp_async16(pf_a + off[j], pf_g + (lane * CH + j) * E);         \
        } else {                                                                  \
          _Pragma("unroll") for (int j = 0; j < CH; ++j) {                        \
            const int cb = (lane * CH + j) * E;                                   \
            if (pt.vec && cb + E <= pt.Lw) {                                      \
              pipe_cp_async16(pf_a + off[j], pf_g + cb);                          \
            } else {                                                              \
              _Pragma("unroll") for (int e = 0; e < E; ++e) if (cb + e < pt.Lw)   \
                  pipe_cp_async(pf_a + off[j] + (uint32_t)(e * sizeof(T)), pf_g + cb + e); \
            }                                                                     \
          }                                                                       \
        }                                                                         \
      }                                                                           \
      pipe_commit();                                                              \
      pipe_wait_group<kPrefetch>();                                               \
      pf_a += RB;                                                                 \
      if (pf_a == in_end) pf_a = ring_in;                                         \
      pf_g += pitch;                                                              \
    }                                                                             \
    load_row_at<CH>(in_a, off, TP2);                                              \
    in_a += RB;                                                                   \
    if (in_a == in_end) in_a = ring_in;                                           \
    if (DTB_PIPE_ROW2) {                                                          \
      row_update2<T, K, DYN>(TM1, TC, TP1, BR, BM3, BM2, BM1, o, wt, lc);         \
    } else {                                                                      \
      row_update<T, K, DYN>(TM1, TC, TP1, BR, wt, lc);                            \
      row_update<T, K, DYN>(BM3, BM2, BM1, o, wt, lc);                            \
    }                                                                             \
    if constexpr (RL == 2) {                                                      \
      if (MIR) mirror_row(r - 2, o);                                              \
      if (r - 2 >= pt.oy0 && r - 2 < pt.oy1) {                                    \
        if (full_vec) {                                                           \
          typedef typename Arith<T>::vec_t V;                                     \
          _Pragma("unroll") for (int j = 0; j < CH; ++j) {                        \
            V x;                                                                  \
            T* px = reinterpret_cast<T*>(&x);                                     \
            _Pragma("unroll") for (int e = 0; e < E; ++e) px[e] = o[j * E + e];   \
            *reinterpret_cast<V*>(st_g + j * E) = x;                              \
          }                                                                       \
        } else {                                                                  \
          _Pragma("unroll") for (int e = 0; e < K; ++e)                           \
              if (c_lo + e >= pt.ox0 && c_lo + e < pt.ox1) st_g[e] = o[e];        \
        }                                                                         \
      }                                                                           \
      st_g += pitch;                                                              \
    } else {                                                                      \
      store_row_at<CH>(out_a, off, o);                                            \
      out_a += RB;                                                                \
      if (out_a == out_end) out_a = ring_out;                                     \
    }                                                                             \
    ++r;                                                                          \
  }
      while (r + 6 < Lh) {
        wait_in(r + 5);
        wait_out(r + 1);
        DTB_PIPE_SPEC_ROW(t3, t0, t1, t2, b0, b3, b2, b1)
        DTB_PIPE_SPEC_ROW(t0, t1, t2, t3, b1, b0, b3, b2)
        DTB_PIPE_SPEC_ROW(t1, t2, t3, t0, b2, b1, b0, b3)
        DTB_PIPE_SPEC_ROW(t2, t3, t0, t1, b3, b2, b1, b0)
        release_in(r);
        release_out(r - 2);
      }
#undef DTB_PIPE_SPEC_ROW
    };
    if (first) steady(std::integral_constant<int, 0>{});
    else if (lastst) steady(std::integral_constant<int, 2>{});
    else steady(std::integral_constant<int, 1>{});
#else
    while (r + 6 < Lh) {
      // one flow-control handshake per 4 rows: inputs r+2..r+5, outputs r-2..r+1
      wait_in(r + 5);
      wait_out(r + 1);
      DTB_PIPE_STEADY(t3, t0, t1, t2, b0, b3, b2, b1)
      DTB_PIPE_STEADY(t0, t1, t2, t3, b1, b0, b3, b2)
      DTB_PIPE_STEADY(t1, t2, t3, t0, b2, b1, b0, b3)
      DTB_PIPE_STEADY(t2, t3, t0, t1, b3, b2, b1, b0)
      release_in(r);       // rows < r are consumed (r+0, r+1 may still be loading)
      release_out(r - 2);  // outputs < r-2 written
    }
#endif
    // tail until every output row is out (r = Lh + 1 is the last iteration)
    while (r <= Lh + 1) {
      DTB_PIPE_ITER(t3, t0, t1, t2, b0, b3, b2, b1)
      if (r > Lh + 1) break;
      DTB_PIPE_ITER(t0, t1, t2, t3, b1, b0, b3, b2)
      if (r > Lh + 1) break;
      DTB_PIPE_ITER(t1, t2, t3, t0, b2, b1, b0, b3)
      if (r > Lh + 1) break;
      DTB_PIPE_ITER(t2, t3, t0, t1, b3, b2, b1, b0)
    }
#undef DTB_PIPE_ITER
#undef DTB_PIPE_STEADY
  }
#if DTB_PIPE_PROBE
  if (lane == 0) {
    atomicAdd(&g_pipe_probe[stage][0], w_in);
    atomicAdd(&g_pipe_probe[stage][1], w_out);
    atomicAdd(&g_pipe_probe[stage][2], clock64() - t_all);
  }
#endif
  if (first) pipe_wait_group<0>();  // drain empty tail groups
  if (!first && lane == 0) st_release_cta(cons + stage, seq0 + Lh);  // whole tile consumed
}

template <typename T, int K, int NW, bool DYN, bool MIR = false>
__device__ __forceinline__ void pipe_stage(const PipeTile& pt, int stage, int nstages, int levels,
                                           int seq0, const T* __restrict__ src,
                                           T* __restrict__ dst, int64_t pitch, uint32_t ring_in,
                                           uint32_t ring_out, int* prod, int* cons,
                                           const Weights<T>& wt, const LaneCtx& lc,
                                           const HaloMirror<T>* mir = nullptr) {
  if (DTB_PIPE_ROLES && stage == 0)
    pipe_stage_role<T, K, NW, DYN, 0, MIR>(pt, stage, levels, seq0, src, dst, pitch, ring_in,
                                           ring_out, prod, cons, wt, lc, nstages, mir);
  else if (DTB_PIPE_ROLES && stage == nstages - 1)
    pipe_stage_role<T, K, NW, DYN, 2, MIR>(pt, stage, levels, seq0, src, dst, pitch, ring_in,
                                           ring_out, prod, cons, wt, lc, nstages, mir);
  else
    pipe_stage_role<T, K, NW, DYN, 1, MIR>(pt, stage, levels, seq0, src, dst, pitch, ring_in,
                                           ring_out, prod, cons, wt, lc, nstages, mir);
}

}  // namespace dtb
