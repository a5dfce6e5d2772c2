/*
 * dtb_b200.h — C ABI of the B200-native deep-temporal-blocking j2d5pt solver.
 *
 * This is the drop-in boundary for the reference's hot path. The reference
 * (arxiv 2306.03336 package `dtb`) is pure Python and has no FFI layer; its
 * boundary is the Python API, which the ctypes host mirror
 * paper_2306_03336_b200/engine.py re-exposes on top of these entry points:
 *
 *   dtb_j2d5pt_f64  replaces  dtb.engine.run_dtb        (pkg/src/dtb/engine.py:305-326)
 *                   and       dtb.oracle.jacobi_reference (pkg/src/dtb/oracle.py:19-34)
 *                   (same padded float64 (ny+2) x (nx+2) C-order buffer, grid.py:126-162;
 *                   same W,E,S,C,N weight order, grid.py:95-123; same valid-region
 *                   freezing, engine.py:26-30; same TrafficReport fields, metrics.py:39-66)
 *   dtb_j2d5pt_f32  fp32 twin (the reference has no fp32 path; BASELINE configs C3a/C3b)
 *   dtb_plan        replaces  dtb.planner.plan_device_tiles (planner.py:188-243) for the
 *                   B200 execution (single-buffer in-place smem model)
 *   dtb_last_error  the message the reference would put in its exception
 *
 * Buffers are caller-owned, row-major, (ny+2) rows of `pitch` elements
 * (pitch >= nx+2); `out` is fully written, ghost ring included (copied from
 * `in`). `in` is never modified. Calls are blocking and externally
 * synchronous (SPEC: one caller at a time per process).
 *
 * Results are bitwise identical to the reference's jacobi_reference: every
 * cell update is ((((W*w + E*e) + S*s) + C*c) + N*n) with every product and
 * sum rounded separately (no FMA). When w, e, s and n are bitwise equal (the
 * reference's StencilWeights.diffusive) the kernels form each source cell's
 * product x*w once and use it for all four neighbours — the same rounded
 * numbers, 6 instead of 9 operations per cell update.
 */
#ifndef DTB_B200_H
#define DTB_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the Python mirror maps them onto the reference's exceptions */
#define DTB_OK 0
#define DTB_EINVAL 1       /* ValueError      (engine.py:236-248, grid.py:111-115) */
#define DTB_ERANGE 2       /* IndexError      (engine.py:249-251, kernel.py:85-91) */
#define DTB_EINFEASIBLE 3  /* InfeasiblePlanError (planner.py:51-56, 222-228) */
#define DTB_ECUDA 4        /* EngineError: CUDA runtime failure (engine.py:49-50) */
#define DTB_ECAPACITY 5    /* EngineError: capacity contract (engine.py:141-145) */

/* flags */
#define DTB_FLAG_POISON 1u          /* NaN-fill scratch that no valid cell may read (engine.py:16-20,174-177) */
#define DTB_FLAG_FORCE_STREAM 2u    /* use the streaming (T-fused HBM pass) kernel even if resident fits */
#define DTB_FLAG_FORCE_NAIVE 4u     /* one global-memory step per launch (the T=1 HBM baseline) */
#define DTB_FLAG_FORCE_DEPTH 8u     /* use t_depth as the temporal halo depth instead of the planner's */
#define DTB_FLAG_TRACE 16u          /* resident kernel: per-CTA clock64 phase counters (dtb_last_trace) */
#define DTB_FLAG_FORCE_PIPE 32u     /* use the pipelined (warp-pipeline, column-strip) streaming kernel */
#define DTB_FLAG_FORCE_RESIDENT 64u /* use the smem-resident kernel (fails if the grid does not fit) */
#define DTB_FLAG_SLAB_COPY 128u     /* n_gpus > 1: exchange slab halos by copies after each epoch */
#define DTB_FLAG_SLAB_FUSED 256u    /* n_gpus > 1: pipelined kernel on every slab, halos stored
                                       into the neighbours in-kernel (fails if a slab cannot) */
#define DTB_FLAG_COUNT 512u         /* report the traffic the kernels COUNTED at their copy and
                                       compute sites (device counters) instead of the schedule's
                                       analytic model; the two agree exactly (tests) */

/* Half-open rectangle in interior coordinates (grid.py:38-92). */
typedef struct dtb_rect {
  int64_t x0, y0, width, height;
} dtb_rect;

/* Cell-granular traffic of the B200 execution (metrics.py:39-66 field order). */
typedef struct dtb_report {
  int64_t global_load_cells;
  int64_t global_store_cells;
  int64_t halo_exchanged_cells;
  int64_t redundant_compute_cells;
  int64_t useful_compute_cells;
  int64_t scratchpad_peak_bytes;
  int64_t elem_bytes;
} dtb_report;

/* The B200 plan (what plan_device_tiles' TilingPlan is for the reference). */
typedef struct dtb_plan_info {
  int32_t mode;         /* 0 resident (persistent, smem-resident), 1 streaming (tile sweep),
                           2 naive, 3 pipelined streaming (warp pipeline) */
  int32_t elem_bytes;
  int32_t lane_elems;   /* K: consecutive columns per lane */
  int32_t warps;        /* warps per CTA (row bands) */
  int32_t halo;         /* temporal halo depth h = steps per exchange / per HBM pass */
  int32_t tiles_x, tiles_y;
  int32_t ctas;         /* grid size of the launch */
  int32_t ctas_per_sm;
  int32_t dyn;          /* 1 if a tile's right frozen column is not lane-aligned */
  int64_t smem_bytes;   /* dynamic shared memory per CTA */
  int64_t tile_w, tile_h;                 /* largest owned tile */
  int64_t load_w, load_h;                 /* largest load region */
  int64_t computed_cells_per_step;        /* lane-cells updated per step, all tiles */
  double est_cells_per_clk;               /* planner cost model */
} dtb_plan_info;

/* Host-buffer entry points (H2D + solve + D2H). t_depth >= 1 is the
 * reference plan's depth: total_steps must be a positive multiple of it
 * (engine.py:238-240). valid may be NULL (whole interior). ilp is accepted for
 * API parity (KernelConfig, kernel.py:33-41) and must be >= 1; it cannot
 * change results. rep may be NULL. n_gpus >= 1: with n_gpus > 1 the library
 * splits the grid into n_gpus y-slabs over the visible devices (round-robin;
 * slabs share a device when fewer are visible), exchanging 16-row halos by
 * device-to-device copies or in-kernel peer stores (NVLink P2P) — bitwise
 * equal to n_gpus = 1, with or without a valid region. The call stays
 * blocking. Multi-pass streaming plans on one GPU overlap the host copies
 * with compute: the input streams in by row blocks while the first passes run
 * as a wavefront over the blocks that arrived, and the result streams out by
 * row blocks as the last passes finish them (same bits; DTB_WAVE_ROWS=0 in
 * the environment turns it off). In, out: pinned host memory lets the copies
 * overlap; pageable memory works too. */
int dtb_j2d5pt_f64(const double* in, double* out, int64_t nx, int64_t ny, int64_t pitch,
                   const double w[5], int64_t total_steps, int64_t t_depth,
                   const dtb_rect* valid, int ilp, int n_gpus, unsigned flags,
                   dtb_report* rep);
int dtb_j2d5pt_f32(const float* in, float* out, int64_t nx, int64_t ny, int64_t pitch,
                   const float w[5], int64_t total_steps, int64_t t_depth,
                   const dtb_rect* valid, int ilp, int n_gpus, unsigned flags,
                   dtb_report* rep);

/* Device-pointer entry points on the current device; `stream` is a
 * cudaStream_t (NULL = legacy default). Asynchronous with respect to the host
 * except for plan/scratch setup; in and out must not alias. Solves share the
 * device's scratch (halo exchange buffers, the streaming ping-pong buffer):
 * solves queued on different streams must be ordered by the caller (one
 * stream, or an event between them). Any origin alignment is accepted; a
 * grid origin off a 16-byte boundary is solved in an aligned staging copy. */
int dtb_j2d5pt_f64_dev(const double* d_in, double* d_out, int64_t nx, int64_t ny,
                       int64_t pitch, const double w[5], int64_t total_steps,
                       int64_t t_depth, const dtb_rect* valid, unsigned flags,
                       void* stream, dtb_report* rep);
int dtb_j2d5pt_f32_dev(const float* d_in, float* d_out, int64_t nx, int64_t ny,
                       int64_t pitch, const float w[5], int64_t total_steps,
                       int64_t t_depth, const dtb_rect* valid, unsigned flags,
                       void* stream, dtb_report* rep);

/* Plan without executing (the B200 analogue of plan_device_tiles). */
int dtb_plan(int64_t nx, int64_t ny, int32_t elem_bytes, int64_t total_steps,
             int64_t t_depth, unsigned flags, dtb_plan_info* out);

/* Phase counters of the most recent DTB_FLAG_TRACE resident solve on this
 * thread: for each CTA, SM clock cycles spent in {compute, publish, wait,
 * refresh}, the epoch count, and the publish split {stores, barrier} (8 values
 * per CTA, the last unused). Copies up to n values into out and returns the
 * number of CTAs (0 if no trace). */
int64_t dtb_last_trace(int64_t* out, int64_t n);

/* Kernel launches issued by the most recent solve on this thread. */
int64_t dtb_last_launch_count(void);

/* After a DTB_EINFEASIBLE: the smallest dynamic shared memory per CTA (bytes)
 * a plan of the requested kind would need — the B200 counterpart of
 * InfeasiblePlanError.min_required_bytes (planner.py:51-56, 222-228). 0 after
 * any other outcome. */
int64_t dtb_last_min_required_bytes(void);

/* Device properties the planner uses (cudaDeviceGetAttribute). */
int dtb_device_info(int32_t* sms, int64_t* smem_optin_per_block, int64_t* l2_bytes,
                    int32_t* cc_major, int32_t* cc_minor);

/* On-device splitmix64 fill, bit-identical to grid_new(nx, ny,
 * random_interior(nx, ny, seed), ghost) (prng.py:45-67, grid.py:165-196). */
int dtb_fill_random_f64(double* d_out, int64_t nx, int64_t ny, int64_t pitch,
                        uint64_t seed, double ghost, void* stream);
int dtb_fill_random_f32(float* d_out, int64_t nx, int64_t ny, int64_t pitch,
                        uint64_t seed, double ghost, void* stream);

/* Rows [row0, row0 + nrows) of that padded grid only, written from d_out's
 * first row (a multi-GPU slab fills its own rows without the full grid). */
int dtb_fill_random_rows_f64(double* d_out, int64_t nx, int64_t ny, int64_t pitch,
                             uint64_t seed, double ghost, int64_t row0, int64_t nrows,
                             void* stream);

/* ---- one process per GPU (multi-process y-slabs, fused halo exchange) ----
 * A slab solver in process r keeps its padded local grid in two buffers
 * allocated with dtb_ipc_malloc and shares their handles with its y-neighbour
 * processes, which map them with dtb_ipc_open. Each epoch's solve then stores
 * the rows the neighbours need straight into the neighbours' buffers from
 * inside the pipelined kernel (NVLink P2P stores between GPUs), and restricts
 * its own stores to the rows it owns: */
typedef struct dtb_halo_mirror {
  void* peer[2];          /* neighbour buffers (this process's mappings), or NULL */
  int64_t r0[2], r1[2];   /* local padded rows [r0, r1) of the result go to peer i ... */
  int64_t p0[2];          /* ... at its rows p0[i] .. (same pitch and column origin) */
  int64_t sw0, sw1;       /* own stores only into local padded rows [sw0, sw1) */
} dtb_halo_mirror;

/* dtb_j2d5pt_*_dev with the fused halo stores of `mir` (the pipelined kernel
 * runs the solve; its last pass writes the mirror rows). total_steps must not
 * exceed the slab's halo depth; the caller orders epochs across processes
 * (dtb_ipc_event_* below). */
int dtb_j2d5pt_f64_dev_mirror(const double* d_in, double* d_out, int64_t nx, int64_t ny,
                              int64_t pitch, const double w[5], int64_t total_steps,
                              const dtb_halo_mirror* mir, void* stream, dtb_report* rep);
int dtb_j2d5pt_f32_dev_mirror(const float* d_in, float* d_out, int64_t nx, int64_t ny,
                              int64_t pitch, const float w[5], int64_t total_steps,
                              const dtb_halo_mirror* mir, void* stream, dtb_report* rep);

/* CUDA IPC: device buffers (cudaMalloc + cudaIpcGetMemHandle) and
 * interprocess events; handles are 64 opaque bytes. */
int dtb_ipc_malloc(int64_t bytes, void** ptr, uint8_t handle[64]);
int dtb_ipc_free(void* ptr);
int dtb_ipc_open(const uint8_t handle[64], void** ptr);
int dtb_ipc_close(void* ptr);
int dtb_ipc_event_create(void** event, uint8_t handle[64]);
int dtb_ipc_event_open(const uint8_t handle[64], void** event);
int dtb_event_destroy(void* event);
int dtb_event_record(void* event, void* stream);
int dtb_stream_wait_event(void* stream, void* event);

/* Last error message on this thread ("" if none). */
const char* dtb_last_error(void);

/* Debug builds only (-DDTB_PIPE_PROBE=1): per pipe stage s, out[3s..3s+2] =
 * {cycles waiting for input rows, cycles waiting for ring space, total cycles}
 * summed over warps since the last call (then reset). DTB_EINVAL otherwise. */
int dtb_debug_pipe_probe(uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* DTB_B200_H */
