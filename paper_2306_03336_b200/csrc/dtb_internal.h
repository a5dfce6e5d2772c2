// dtb_internal.h — declarations shared by the library's translation units
// (host runtime dtb_host.cu, the kernel TUs dtb_resident_*.cu, dtb_pipe_*.cu,
// dtb_stream.cu, and the planner dtb_plan.cpp). Not part of the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/dtb_b200.h"
#include "dtb_plan.h"

namespace dtb {

template <typename T> struct Weights;

constexpr int kMaxTiles = 512;  // per dimension
constexpr int kMaxWaveTasks = 72;  // (pass, row block) tasks per wavefront diagonal

// Tile geometry as kernel parameters (<= 32 KB param space on sm_70+ / CUDA 12.1+).
// col[i] = (owned x0, owned x1, load x0, load x1) in interior coordinates.
struct Geometry {
  int ntx, nty;
  int4 col[kMaxTiles];
  int4 row[kMaxTiles];
};

// Fused slab halo exchange (n_gpus > 1): the pipelined kernel's last stage
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

// ---- per-thread call state (the C ABI is externally synchronous) ----------
extern thread_local std::string g_err;
extern thread_local int64_t g_launches;
extern thread_local std::vector<int64_t> g_trace;
extern thread_local unsigned g_flags;
// set by the slab drivers around one slab's solve: the pipe kernel's final
// pass then feeds the neighbour slabs' halos in-kernel (HaloMirror)
extern thread_local const void* g_halo_mirror;
// planner minimum for the last DTB_EINFEASIBLE (InfeasiblePlanError.min_required_bytes)
extern thread_local int64_t g_min_bytes;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return ::dtb::fail(DTB_ECUDA, "CUDA error %s (%s) at %s:%d", cudaGetErrorName(e_), \
                         cudaGetErrorString(e_), __FILE__, __LINE__);                    \
  } while (0)

// Per-device scratch, grown on demand and kept (solves are externally
// synchronous, so one arena per device and role suffices).
enum ArenaRole { kArenaScratch = 0, kArenaIo = 1, kArenaStage = 2, kArenaCounters = 3,
                 kArenaCount = 4 };
int arena_get(int role, int device, size_t bytes, void** out);

int query_dev(DevInfo& d);
// raise a kernel's dynamic-smem attribute (monotonic, cached) and query its
// occupancy (cached) when per_sm is non-null
int prepare_kernel(const void* kern, int device, int smem, int threads, int* per_sm);

// ---- kernel launchers (one translation unit per family and type) ----------
// cnt (DTB_FLAG_COUNT, else null): device counters the kernels add their
// counted traffic to — [0] global loads, [1] global stores, [2] halo cells
// exchanged, [3] cell updates performed (domain cells; the ghost ring is
// never counted, metrics.py:3-6)
template <typename T>
int launch_resident(const Plan& p, const Geometry& geo, const T* d_in, T* d_out, int64_t pitch,
                    int nx, int ny, const T w[5], int64_t steps, bool poison, cudaStream_t st,
                    unsigned long long* cnt);
template <typename T>
int launch_stream(const Plan& p, const Geometry& geo, const T* d_in, T* d_out, int64_t pitch,
                  int nx, int ny, const T w[5], int64_t steps, bool poison, cudaStream_t st,
                  unsigned long long* cnt);
template <typename T>
int launch_pipe(const Plan& p, const Geometry& geo, const T* d_in, T* d_out, int64_t pitch,
                int nx, int ny, const T w[5], int64_t steps, cudaStream_t st,
                unsigned long long* cnt);
// launch_pipe_wave (dtb_pipe.cuh): in_ready(j) before a launch that reads
// input row blocks <= j, out_done(j) after the launch that finishes output
// row block j (host copies go between); a nonzero return aborts
struct PipeWaveHooks {
  void* ctx;
  int (*in_ready)(void* ctx, int j);
  int (*out_done)(void* ctx, int j);
};
template <typename T>
int launch_pipe_wave(const Plan& p, const Geometry& geo, const Geometry& gw, const T* d_in,
                     T* d_out, int64_t pitch, int nx, int ny, const T w[5], int64_t steps,
                     int64_t m, cudaStream_t st, unsigned long long* cnt,
                     const PipeWaveHooks& hooks);
template <typename T>
int launch_naive(const T* d_in, T* d_out, T* d_tmp, int64_t pitch, int nx, int ny, const T w[5],
                 int64_t steps, cudaStream_t st);
template <typename T>
int launch_fill(T* d_out, int64_t pitch, int nx, int ny, uint64_t seed, double ghost,
                int64_t row0, int64_t nrows, cudaStream_t st);

// w, e, s, n bitwise equal: the kernels' 6-op shared-product form applies
template <typename T>
bool weights_isotropic(const T w[5]);

}  // namespace dtb
