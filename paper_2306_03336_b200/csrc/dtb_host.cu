// dtb_host.cu — host runtime and the C ABI (include/dtb_b200.h).
//
// solve_dev: argument contract (engine.py:236-251), valid-region handling
// (engine.py:26-30), the B200 plan (dtb_plan.cpp) and dispatch to a kernel
// family (dtb_resident_*.cu, dtb_pipe_*.cu, dtb_stream.cu). solve_host_slabs:
// n_gpus > 1 y-slabs with depth-16 halos. The C entry points
// wrap these with host<->device copies.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "dtb_internal.h"

namespace dtb {

thread_local std::string g_err;
thread_local int64_t g_launches = 0;
thread_local std::vector<int64_t> g_trace;
thread_local unsigned g_flags = 0;
thread_local const void* g_halo_mirror = nullptr;
thread_local int64_t g_min_bytes = 0;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

namespace {
struct Arena {
  void* p = nullptr;
  size_t n = 0;
};
std::mutex g_arena_mu;
Arena g_arenas[kArenaCount][16];
}  // namespace

int arena_get(int role, int device, size_t bytes, void** out) {
  std::lock_guard<std::mutex> lk(g_arena_mu);
  Arena& a = g_arenas[role][device & 15];
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
static int query_dev_uncached(DevInfo& d, int dev) {
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

template <typename T>
bool weights_isotropic(const T w[5]) {
  uint64_t b[5] = {0, 0, 0, 0, 0};
  for (int i = 0; i < 5; ++i) memcpy(&b[i], &w[i], sizeof(T));
  return b[0] == b[1] && b[0] == b[2] && b[0] == b[4];
}
template bool weights_isotropic<double>(const double*);
template bool weights_isotropic<float>(const float*);

}  // namespace dtb

// ===========================================================================
namespace {

using namespace dtb;

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

// ---------------------------------------------------------------------------
// TrafficReport of the B200 schedule (metrics.py:39-66 fields, cell units,
// ghost ring never counted, metrics.py:3-6). fill_report is the analytic
// model; with DTB_FLAG_COUNT the kernels count the same quantities at their
// copy and compute sites instead (device counters, dtb_internal.h), and the
// tests require the two to agree exactly:
//   loads   cells read from global memory into shared memory (tile loads,
//           resident halo refreshes from the L2 exchange buffer)
//   stores  cells written back (owned cells, resident halo publishes)
//   halo    cells exchanged between CTAs (refreshes) or slabs (mirror stores)
//   redundant = cell updates performed (every level's rows of every band or
//           segment, frozen rows/columns excluded) - useful
// ---------------------------------------------------------------------------
int64_t span(int64_t a, int64_t b, int64_t lo, int64_t hi) {
  return std::max<int64_t>(0, std::min(b, hi) - std::max(a, lo));
}

void band_rows_host(int Lh, int nb, int b, int& ya, int& yb) {  // dtb_core.cuh band_rows
  const int rows = Lh - 2;
  const int base = rows / nb, rem = rows % nb;
  ya = 1 + b * base + std::min(b, rem);
  yb = ya + base + (b < rem ? 1 : 0);
}

// cell updates of advance_tile over `steps` (dtb_core.cuh: two-step sweeps
// update 2H + 2 rows per band, minus frozen rows; one-step sweeps H)
int64_t sweep_cells(int Lw, int Lh, int steps, int nw, bool poison) {
  const int rows = Lh - 2;
  if (rows <= 0 || Lw <= 2 || steps <= 0) return 0;
  if (poison) return (int64_t)steps * rows * (Lw - 2);
  int64_t c = 0;
  int s = 0;
  if (steps >= 2 && rows >= 2) {
    const int nb = std::max(1, std::min(nw, rows / 2));
    int64_t per = 0;
    for (int b = 0; b < nb; ++b) {
      int ya, yb;
      band_rows_host(Lh, nb, b, ya, yb);
      per += 2 * (yb - ya) + 2 - (ya == 1) - (yb == Lh - 1);
    }
    s = steps / 2 * 2;
    c += (int64_t)(steps / 2) * per * (Lw - 2);
  }
  c += (int64_t)(steps - s) * rows * (Lw - 2);
  return c;
}

template <typename T>
void fill_report(const Plan& p, int64_t nx, int64_t ny, int64_t steps, bool poison,
                 const HaloMirror<T>* mir, dtb_report* rep) {
  if (!rep) return;
  memset(rep, 0, sizeof *rep);
  rep->elem_bytes = (int64_t)sizeof(T);
  rep->useful_compute_cells = nx * ny * steps;
  rep->scratchpad_peak_bytes = p.smem_bytes;
  int64_t load = 0, store = 0, halo = 0, comp = 0;
  if (p.mode == 2) {  // naive: every step reads and writes the grid once
    rep->global_load_cells = rep->global_store_cells = nx * ny * steps;
    rep->scratchpad_peak_bytes = 0;
    return;
  }
  const int ntx = p.sx.n, nty = p.sy.n;
  auto tile = [&](int i, int j, int& Lw, int& Lh, int& gx0, int& gy0) {
    Lw = p.sx.l1[i] - p.sx.l0[i];
    Lh = p.sy.l1[j] - p.sy.l0[j];
    gx0 = p.sx.l0[i] + 1;
    gy0 = p.sy.l0[j] + 1;
  };
  if (p.mode == 0) {  // resident (dtb_resident.cuh)
    const int64_t E = (steps + p.h - 1) / p.h;
    for (int j = 0; j < nty; ++j)
      for (int i = 0; i < ntx; ++i) {
        int Lw, Lh, gx0, gy0;
        tile(i, j, Lw, Lh, gx0, gy0);
        const int cz = p.sx.l0[i], cw = p.sx.l1[i], rz = p.sy.l0[j], rw = p.sy.l1[j];
        const int ox0 = p.sx.o0[i] - cz, ox1 = p.sx.o1[i] - cz;
        const int oy0 = p.sy.o0[j] - rz, oy1 = p.sy.o1[j] - rz;
        const bool hl = cz > -1, hr = cw < nx + 1, ht = rz > -1, hb = rw < ny + 1;
        const int bl = i > 0 ? std::max(0, p.sx.l1[i - 1] - p.sx.o0[i]) : 0;
        const int br = i + 1 < ntx ? std::max(0, p.sx.o1[i] - p.sx.l0[i + 1]) : 0;
        const int bt = j > 0 ? std::max(0, p.sy.l1[j - 1] - p.sy.o0[j]) : 0;
        const int bb = j + 1 < nty ? std::max(0, p.sy.o1[j] - p.sy.l0[j + 1]) : 0;
        const int rx0 = hl ? 0 : 1, rx1 = hr ? Lw : Lw - 1, ry0 = ht ? 0 : 1, ry1 = hb ? Lh : Lh - 1;
        load += span(gy0, gy0 + Lh, 1, ny + 1) * span(gx0, gx0 + Lw, 1, nx + 1);
        store += (int64_t)(oy1 - oy0) * (ox1 - ox0);
        // refresh_flat's ring, by owning neighbour (dtb_tile_io.cuh)
        int64_t refresh = 0;
        const int reg[8][6] = {{0, -1, ry0, oy0, ox0, ox1}, {0, 1, oy1, ry1, ox0, ox1},
                               {-1, -1, ry0, oy0, rx0, ox0}, {1, -1, ry0, oy0, ox1, rx1},
                               {-1, 1, oy1, ry1, rx0, ox0}, {1, 1, oy1, ry1, ox1, rx1},
                               {-1, 0, oy0, oy1, rx0, ox0}, {1, 0, oy0, oy1, ox1, rx1}};
        for (const auto& r : reg) {
          const int nxt = i + r[0], nyt = j + r[1];
          if (r[3] <= r[2] || r[5] <= r[4] || nxt < 0 || nxt >= ntx || nyt < 0 || nyt >= nty) continue;
          refresh += (int64_t)(r[3] - r[2]) * (r[5] - r[4]);
        }
        // the publish of every non-final epoch
        int64_t publish = 0;
        const int owned_w = ox1 - ox0, top1 = oy0 + bt, bot0 = oy1 - bb;
        const int cr0 = std::max(ox1 - br, ox0 + bl), wl = bl, wr = ox1 - cr0;
        if (poison) {
          const int t1 = std::min(oy0 + bt, oy1), b0 = std::max(oy1 - bb, t1);
          publish = (int64_t)(t1 - oy0 + oy1 - b0) * owned_w + (int64_t)(b0 - t1) * (wl + wr);
        } else {
          const int rows = Lh - 2;
          const bool two = p.h >= 2 && rows >= 2 && p.h % 2 == 0;
          const int nb = two ? std::max(1, std::min(p.warps, rows / 2))
                             : std::max(1, std::min(p.warps, rows));
          for (int b = 0; b < nb && rows > 0 && Lw > 2; ++b) {
            int ya, yb;
            band_rows_host(Lh, nb, b, ya, yb);
            const int r0 = std::max(ya, oy0), r1 = std::min(yb, oy1);
            const int s0 = std::max(r0, top1), s1 = std::min(r1, bot0);
            publish += (int64_t)std::max(0, s1 - s0) * (wl + wr) +
                       (int64_t)(std::max(0, std::min(r1, top1) - r0) +
                                 std::max(0, r1 - std::max(r0, bot0))) * owned_w;
          }
        }
        load += (E - 1) * refresh;
        halo += (E - 1) * refresh;
        store += (E - 1) * publish;
        for (int64_t e = 0; e < E; ++e)
          comp += sweep_cells(Lw, Lh, (int)std::min<int64_t>(p.h, steps - e * p.h), p.warps, poison);
      }
  } else {  // streaming passes: pipelined (mode 3) or tile sweep (mode 1)
    const int64_t passes = (steps + p.h - 1) / p.h;
    for (int64_t k = 0; k < passes; ++k) {
      const int s_k = (int)std::min<int64_t>(p.h, steps - k * p.h);
      const bool mirror_pass = mir && k + 1 == passes;
      for (int j = 0; j < nty; ++j)
        for (int i = 0; i < ntx; ++i) {
          int Lw, Lh, gx0, gy0;
          tile(i, j, Lw, Lh, gx0, gy0);
          load += span(gy0, gy0 + Lh, 1, ny + 1) * span(gx0, gx0 + Lw, 1, nx + 1);
          if (p.mode == 3) {  // dtb_pipe.cuh store window and mirror rows
            const int cz = p.sx.l0[i], rz = p.sy.l0[j];
            const int ox0 = p.sx.o0[i] - (p.sx.o0[i] == 0) - cz;
            const int ox1 = p.sx.o1[i] + (p.sx.o1[i] == nx) - cz;
            int oy0 = p.sy.o0[j] - (p.sy.o0[j] == 0) - rz;
            int oy1 = p.sy.o1[j] + (p.sy.o1[j] == ny) - rz;
            const int qy0 = oy0, qy1 = oy1;
            if (mirror_pass) {
              oy0 = std::max<int64_t>(oy0, mir->sw0 - gy0);
              oy1 = std::min<int64_t>(oy1, mir->sw1 - gy0);
            }
            const int64_t sc = span(gx0 + ox0, gx0 + ox1, 1, nx + 1);
            store += span(gy0 + oy0, gy0 + oy1, 1, ny + 1) * sc;
            if (mirror_pass)
              for (int m = 0; m < 2; ++m) halo += span(gy0 + qy0, gy0 + qy1, mir->r0[m], mir->r1[m]) * sc;
            comp += (int64_t)s_k * std::max(0, Lh - 2) * std::max(0, Lw - 2);
          } else {
            store += (int64_t)(p.sy.o1[j] - p.sy.o0[j]) * (p.sx.o1[i] - p.sx.o0[i]);
            comp += sweep_cells(Lw, Lh, s_k, p.warps, poison);
          }
        }
    }
  }
  rep->global_load_cells = load;
  rep->global_store_cells = store;
  rep->halo_exchanged_cells = halo;
  rep->redundant_compute_cells = comp - nx * ny * steps;
}

int plan_fail(const char* err, int64_t min_bytes) {
  g_min_bytes = min_bytes;
  return fail(DTB_EINFEASIBLE, "%s", err);
}

int force_mode(unsigned flags) {
  return (flags & DTB_FLAG_FORCE_NAIVE) ? 2 : (flags & DTB_FLAG_FORCE_STREAM) ? 1
         : (flags & DTB_FLAG_FORCE_PIPE) ? 3 : (flags & DTB_FLAG_FORCE_RESIDENT) ? 4 : 0;
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
  const size_t row_bytes = (size_t)(nx + 2) * sizeof(T);
  // valid-region runs: frozen cells outside `valid` are carried by a copy of
  // the (nx+2)-column grid (never the pitch padding beyond it), and the valid
  // rectangle evolves as a standalone problem whose ghost ring is the
  // surrounding frozen cells (engine.py:26-30, grid.py:199-222).
  int64_t vx = 0, vy = 0, vnx = nx, vny = ny;
  if (valid && !(valid->x0 == 0 && valid->y0 == 0 && valid->width == nx && valid->height == ny)) {
    CUDA_TRY(cudaMemcpy2DAsync(d_out, pitch * sizeof(T), d_in, pitch * sizeof(T), row_bytes,
                               ny + 2, cudaMemcpyDeviceToDevice, st));
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
    if (int rc2 = arena_get(kArenaStage, device, 2 * sbytes, &sp)) return rc2;
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
  const int depth = (flags & DTB_FLAG_FORCE_DEPTH) ? (int)t_depth : 0;
  Plan p;
  char err[512];
  int64_t min_bytes = 0;
  if (!make_plan(vnx, vny, (int)sizeof(T), total_steps, dev, force_mode(flags), depth, p, err,
                 sizeof err, &min_bytes))
    return plan_fail(err, min_bytes);
  const bool poison = (flags & DTB_FLAG_POISON) != 0;
  if (g_halo_mirror && p.mode != 3)
    return fail(DTB_EINVAL, "fused slab halos need the pipelined kernel (plan mode %d)", p.mode);
  // DTB_FLAG_COUNT: the kernels count their traffic into device counters
  unsigned long long* cnt = nullptr;
  if ((flags & DTB_FLAG_COUNT) && p.mode != 2) {
    int device;
    CUDA_TRY(cudaGetDevice(&device));
    void* c = nullptr;
    if (int rc2 = arena_get(kArenaCounters, device, 8 * sizeof(unsigned long long), &c)) return rc2;
    cnt = static_cast<unsigned long long*>(c);
    CUDA_TRY(cudaMemsetAsync(cnt, 0, 8 * sizeof(unsigned long long), st));
  }
  if (p.mode == 2) {
    // naive: total_steps launches ping-ponging between out and scratch
    const size_t grid_bytes = (size_t)(ny + 2) * pitch * sizeof(T);
    T* tmp = nullptr;
    if (total_steps > 1) {
      void* s = nullptr;
      int device;
      CUDA_TRY(cudaGetDevice(&device));
      if (int rc2 = arena_get(kArenaScratch, device, grid_bytes, &s)) return rc2;
      tmp = reinterpret_cast<T*>(s);
      if (valid)  // the frozen cells around the window, in the scratch parity too
        CUDA_TRY(cudaMemcpy2DAsync(tmp, pitch * sizeof(T), d_in, pitch * sizeof(T), row_bytes,
                                   ny + 2, cudaMemcpyDeviceToDevice, st));
    }
    T* tmp_v = tmp ? tmp + vy * pitch + vx : nullptr;
    rc = launch_naive<T>(in_v, out_v, tmp_v, pitch, (int)vnx, (int)vny, w, total_steps, st);
    if (rc) return rc;
  } else {
    Geometry geo;
    rc = fill_geometry(p, geo);
    if (rc) return rc;
    if (p.mode == 0)
      rc = launch_resident<T>(p, geo, in_v, out_v, pitch, (int)vnx, (int)vny, w, total_steps,
                              poison, st, cnt);
    else if (p.mode == 3)
      rc = launch_pipe<T>(p, geo, in_v, out_v, pitch, (int)vnx, (int)vny, w, total_steps, st, cnt);
    else
      rc = launch_stream<T>(p, geo, in_v, out_v, pitch, (int)vnx, (int)vny, w, total_steps,
                            poison, st, cnt);
    if (rc) return rc;
  }
  fill_report<T>(p, vnx, vny, total_steps, poison, static_cast<const HaloMirror<T>*>(g_halo_mirror),
                 rep);
  if (cnt && rep) {  // replace the model by what the kernels counted
    unsigned long long h[8];
    CUDA_TRY(cudaMemcpyAsync(h, cnt, sizeof h, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    rep->global_load_cells = (int64_t)h[0];
    rep->global_store_cells = (int64_t)h[1];
    rep->halo_exchanged_cells = (int64_t)h[2];
    rep->redundant_compute_cells = (int64_t)h[3] - vnx * vny * total_steps;
  }
  return DTB_OK;
}

// ---------------------------------------------------------------------------
// n_gpus > 1 from the host entry: y-slabs (the native twin of
// slab.py). Slab g owns interior rows [y0, y1) and keeps a local padded grid
// of those rows plus kSlabDepth halo rows towards each neighbour (the global
// ghost row on the outer sides). Every epoch of s <= depth steps each slab
// advances its local grid s steps with its outer rows frozen (the trapezoid
// argument: owned rows stay exact), then receives depth rows from each
// neighbour into its halo. Slabs go round-robin over the visible devices;
// slabs sharing a device run in order on that device's stream, so no kernel
// ever waits on another's. Bitwise equal to n_gpus = 1.
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

// Peer access between two devices, enabled once. Usable only when enabling
// succeeded or it was already enabled; any other failure (e.g. too many
// peers) means in-kernel stores to the peer would fault, so callers fall
// back to copies.
bool peer_usable(int from, int to) {
  if (from == to) return true;
  static std::mutex mu;
  static int state[16][16] = {};  // 0 unknown, 1 usable, 2 not usable
  std::lock_guard<std::mutex> lk(mu);
  int& s = state[from & 15][to & 15];
  if (s == 0) {
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, from, to) != cudaSuccess) can = 0;
    s = 2;
    if (can) {
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(from);
      const cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
      if (e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled) s = 1;
      cudaGetLastError();  // clear a non-sticky enable error
      cudaSetDevice(cur);
    }
  }
  return s == 1;
}

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
  auto devof = [&](int d) { return (dev0 + d) % ndev; };
  for (int d = 0; d < (int)dstream.size(); ++d) {
    CUDA_TRY(cudaSetDevice(devof(d)));
    CUDA_TRY(cudaStreamCreateWithFlags(&dstream[d], cudaStreamNonBlocking));
    res.streams.push_back({devof(d), dstream[d]});
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
    CUDA_TRY(cudaSetDevice(devof(s.dev)));
    void* p = nullptr;
    CUDA_TRY(cudaMalloc(&p, 2 * bytes));
    res.bufs.push_back({devof(s.dev), p});
    s.a = reinterpret_cast<T*>(p);
    s.b = reinterpret_cast<T*>(reinterpret_cast<char*>(p) + bytes);
    CUDA_TRY(cudaMemcpy2DAsync(s.a, drow, in + s.row0 * pitch, pitch * sizeof(T), hrow,
                               s.lny + 2, cudaMemcpyHostToDevice, dstream[s.dev]));
  }
  // exchange mode: fused (the pipe kernel's final pass of each epoch stores
  // the neighbours' halo rows straight into their next input, P2P when they
  // live on another GPU) whenever every slab runs the pipelined kernel and
  // every neighbour pair has usable peer access; else device-to-device
  // copies after each epoch
  bool fused = (flags & DTB_FLAG_SLAB_COPY) == 0 && n_slabs > 1;
  for (int g = 0; g + 1 < n_slabs && fused; ++g) {
    const int da = devof(sl[g].dev), db = devof(sl[g + 1].dev);
    fused = peer_usable(da, db) && peer_usable(db, da);
  }
  if (n_slabs > 1 && !fused) {  // best effort: direct NVLink copies
    for (int g = 0; g + 1 < n_slabs; ++g) {
      const int da = devof(sl[g].dev), db = devof(sl[g + 1].dev);
      peer_usable(da, db);
      peer_usable(db, da);
    }
  }
  CUDA_TRY(cudaSetDevice(dev0));
  if (fused) {
    DevInfo di;
    if (int rc = query_dev(di)) return rc;
    const int force = (flags & DTB_FLAG_SLAB_FUSED) ? 3 : 0;
    for (int g = 0; g < n_slabs && fused; ++g) {
      Plan p;
      char err[256];
      fused = make_plan(nx, sl[g].lny, (int)sizeof(T), depth, di, force, 0, p, err, sizeof err,
                        nullptr) &&
              p.mode == 3;
    }
  }
  if ((flags & DTB_FLAG_SLAB_FUSED) && !fused)
    return fail(DTB_EINFEASIBLE, "fused slab halos need the pipelined kernel and peer access on every slab");
  std::vector<cudaEvent_t> solved(2 * n_slabs), copied(n_slabs);  // solved: epoch parity
  for (int g = 0; g < n_slabs; ++g) {
    CUDA_TRY(cudaSetDevice(devof(sl[g].dev)));
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
      CUDA_TRY(cudaSetDevice(devof(s.dev)));
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
        // the last epoch feeds no one: plain solve (its halo rows are never read)
        const bool final_epoch = done + s_ep >= total_steps;
        MirrorScope scope(fused && !final_epoch ? &m : nullptr);
        if (int rc = solve_dev<T>(s.a, s.b, nx, s.lny, dpitch, w, s_ep, 1, nullptr, lflags, st, &r))
          return rc;
      }
      launches += g_launches;
      acc.global_load_cells += r.global_load_cells;
      acc.global_store_cells += r.global_store_cells;
      acc.halo_exchanged_cells += r.halo_exchanged_cells;  // fused: the mirror stores
      acc.redundant_compute_cells += r.redundant_compute_cells + r.useful_compute_cells;
      acc.scratchpad_peak_bytes = std::max(acc.scratchpad_peak_bytes, r.scratchpad_peak_bytes);
      std::swap(s.a, s.b);
      CUDA_TRY(cudaEventRecord(solved[cur * n_slabs + g], st));
    }
    done += s_ep;
    ++epoch;
    if (done >= total_steps) break;
    if (fused) continue;
    for (int g = 0; g < n_slabs; ++g) {  // halo rows from each neighbour's owned edge rows
      Slab& s = sl[g];
      cudaStream_t st = dstream[s.dev];
      CUDA_TRY(cudaSetDevice(devof(s.dev)));
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
    CUDA_TRY(cudaSetDevice(devof(s.dev)));
    const int64_t r0 = g == 0 ? 0 : s.ht, r1 = s.ht + s.own + (g + 1 == n_slabs ? 1 : 0);
    CUDA_TRY(cudaMemcpy2DAsync(out + (s.row0 + r0) * pitch, pitch * sizeof(T), s.a + r0 * dpitch,
                               drow, hrow, r1 - r0, cudaMemcpyDeviceToHost, dstream[s.dev]));
  }
  for (int d = 0; d < (int)dstream.size(); ++d) {
    CUDA_TRY(cudaSetDevice(devof(d)));
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

// ---------------------------------------------------------------------------
// Host-buffer solves of streaming plans: the passes run as a temporal
// wavefront over row blocks (launch_pipe_wave) so that the host copies
// overlap compute. The input is copied block by block on a copy stream and
// each diagonal waits only for the blocks its first-pass tasks read; each
// final row block is copied back as soon as its last-pass task's diagonal is
// done. Without this the PCIe copies of C4 (2 x 2.15 GB) sit serially around
// 125 passes.
// ---------------------------------------------------------------------------
namespace {

struct WaveStreams {  // per device, created once (the C ABI is externally synchronous)
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> ev;
};
WaveStreams g_wave[64];

template <typename T>
struct WaveCopies {
  const T* in;
  T* out;
  T* d_in;
  T* d_out;
  int64_t pitch, dpitch, nx, ny;
  int J;
  std::vector<int64_t> r0, r1;  // padded rows of row block j (ghost rows at the ends)
  cudaStream_t st, h2d, d2h;
  cudaEvent_t* ev;              // [0, J): input block landed; [J, 2J): output block final
  int waited = -1;
};

template <typename T>
int wave_in_ready(void* c, int j) {  // the next launch reads input row blocks <= j
  WaveCopies<T>& w = *static_cast<WaveCopies<T>*>(c);
  if (j > w.waited) {
    CUDA_TRY(cudaStreamWaitEvent(w.st, w.ev[j], 0));
    w.waited = j;
  }
  return DTB_OK;
}

template <typename T>
int wave_out_done(void* c, int j) {  // output row block j is final once `st` gets here
  WaveCopies<T>& w = *static_cast<WaveCopies<T>*>(c);
  cudaEvent_t e = w.ev[w.J + j];
  CUDA_TRY(cudaEventRecord(e, w.st));
  CUDA_TRY(cudaStreamWaitEvent(w.d2h, e, 0));
  const size_t row = (size_t)(w.nx + 2) * sizeof(T);
  CUDA_TRY(cudaMemcpy2DAsync(w.out + w.r0[j] * w.pitch, w.pitch * sizeof(T),
                             w.d_out + w.r0[j] * w.dpitch, w.dpitch * sizeof(T), row,
                             w.r1[j] - w.r0[j], cudaMemcpyDeviceToHost, w.d2h));
  return DTB_OK;
}

// rows per wavefront row block (DTB_WAVE_ROWS, 0 = off): more blocks overlap
// more of the copies, each block adds 2h rows of pass halo
int64_t wave_rows() {
  const char* e = getenv("DTB_WAVE_ROWS");
  return e ? atoll(e) : 192;
}

// passes per wavefront phase: ~3/4 of the passes the host copy of the grid
// takes (PCIe ~50 GB/s against ~1.35 / 1.9 Tcells/s per fp64 / fp32 pass).
// B200, C4 e2e (profiles/r02/ab_wave*.log): 192-row blocks with 20 passes
// 1142 GCells/s, 26 -> 1131, 32 -> 1117, 10 -> 1069; 128 / 256 rows 1128 /
// 1118; no wavefront 979.
int64_t wave_passes(int64_t nx, int64_t ny, int elem, int64_t passes) {
  if (const char* e = getenv("DTB_WAVE_PASSES")) return std::max<int64_t>(1, atoll(e));
  const double copy_s = (double)(nx + 2) * (ny + 2) * elem / 50e9;
  const double pass_s = (double)nx * ny * 8 / (elem == 8 ? 1.35e12 : 1.9e12);
  return std::min<int64_t>(passes, (int64_t)std::ceil(0.75 * copy_s / pass_s));
}

}  // namespace

// returns DTB_OK after a wavefront solve, -1 when the plan is not a
// multi-pass streaming plan (the caller solves the plain way)
template <typename T>
int solve_host_wave(const T* in, T* out, int64_t nx, int64_t ny, int64_t pitch, const T w[5],
                    int64_t total_steps, unsigned flags, dtb_report* rep) {
  const int64_t rows = wave_rows();
  if (rows <= 0 || g_halo_mirror ||
      (flags & (DTB_FLAG_POISON | DTB_FLAG_TRACE | DTB_FLAG_FORCE_STREAM | DTB_FLAG_FORCE_NAIVE |
                DTB_FLAG_FORCE_RESIDENT | DTB_FLAG_FORCE_DEPTH)))
    return -1;
  DevInfo dev;
  if (int rc = query_dev(dev)) return rc;
  Plan p;
  char err[512];
  int64_t min_bytes = 0;
  if (!make_plan(nx, ny, (int)sizeof(T), total_steps, dev, force_mode(flags), 0, p, err,
                 sizeof err, &min_bytes))
    return plan_fail(err, min_bytes);
  const int64_t passes = (total_steps + p.h - 1) / p.h;
  if (p.mode != 3 || passes < 2) return -1;
  // a diagonal carries about J / 2 row-block tasks of ntx strips each; unless
  // that fills the device's pipelines twice over (narrow grids, e.g. C3b's 35
  // strips) the wavefront costs more than the copies it hides
  const int64_t pipes = (int64_t)dev.sms * (p.warps / 4);
  const int J = (int)std::min<int64_t>(2 * kMaxWaveTasks - 2, std::max<int64_t>(2, ny / rows));
  if (!getenv("DTB_WAVE_ROWS") && (int64_t)(J / 2) * p.sx.n < 2 * pipes) return -1;
  Split sy;
  int nj = J;
  for (; nj >= 2; --nj)
    if (make_split((int)ny, nj, p.h, 1, 1 << 30, p.h, sy)) break;
  if (nj < 2) return -1;
  Plan pw = p;  // the wavefront phases' row blocks
  pw.sy = sy;
  Geometry geo, gw;
  if (int rc = fill_geometry(p, geo)) return rc;
  if (int rc = fill_geometry(pw, gw)) return rc;
  const int64_t m = wave_passes(nx, ny, (int)sizeof(T), passes);
  int device;
  CUDA_TRY(cudaGetDevice(&device));
  if (device < 0 || device >= 64) return -1;
  WaveStreams& ws = g_wave[device];
  if (!ws.h2d) {
    CUDA_TRY(cudaStreamCreateWithFlags(&ws.h2d, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&ws.d2h, cudaStreamNonBlocking));
  }
  while ((int)ws.ev.size() < 2 * nj) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ws.ev.push_back(e);
  }
  const int64_t dpitch = (nx + 2 + 31) / 32 * 32;
  const size_t bytes = (size_t)(ny + 2) * dpitch * sizeof(T);
  void* io = nullptr;
  if (int rc = arena_get(kArenaIo, device, 2 * bytes, &io)) return rc;
  WaveCopies<T> c;
  c.in = in;
  c.out = out;
  c.d_in = reinterpret_cast<T*>(io);
  c.d_out = reinterpret_cast<T*>(reinterpret_cast<char*>(io) + bytes);
  c.pitch = pitch;
  c.dpitch = dpitch;
  c.nx = nx;
  c.ny = ny;
  c.J = nj;
  c.st = 0;
  c.h2d = ws.h2d;
  c.d2h = ws.d2h;
  c.ev = ws.ev.data();
  for (int j = 0; j < nj; ++j) {
    c.r0.push_back(j == 0 ? 0 : sy.o0[j] + 1);
    c.r1.push_back(j == nj - 1 ? ny + 2 : sy.o1[j] + 1);
  }
  g_launches = 0;
  g_flags = flags;
  g_trace.clear();
  // the copy stream starts after earlier work on the solve stream (arena reuse)
  CUDA_TRY(cudaEventRecord(ws.ev[0], c.st));
  CUDA_TRY(cudaStreamWaitEvent(c.h2d, ws.ev[0], 0));
  CUDA_TRY(cudaStreamWaitEvent(c.d2h, ws.ev[0], 0));
  const size_t row = (size_t)(nx + 2) * sizeof(T);
  for (int j = 0; j < nj; ++j) {
    CUDA_TRY(cudaMemcpy2DAsync(c.d_in + c.r0[j] * dpitch, dpitch * sizeof(T), in + c.r0[j] * pitch,
                               pitch * sizeof(T), row, c.r1[j] - c.r0[j], cudaMemcpyHostToDevice,
                               c.h2d));
    CUDA_TRY(cudaEventRecord(ws.ev[j], c.h2d));
  }
  unsigned long long* cnt = nullptr;
  if (flags & DTB_FLAG_COUNT) {
    void* cp = nullptr;
    if (int rc = arena_get(kArenaCounters, device, 8 * sizeof(unsigned long long), &cp)) return rc;
    cnt = static_cast<unsigned long long*>(cp);
    CUDA_TRY(cudaMemsetAsync(cnt, 0, 8 * sizeof(unsigned long long), c.st));
  }
  PipeWaveHooks hooks{&c, wave_in_ready<T>, wave_out_done<T>};
  int rc = launch_pipe_wave<T>(p, geo, gw, c.d_in, c.d_out, dpitch, (int)nx, (int)ny, w,
                               total_steps, m, c.st, cnt, hooks);
  // drain both copy streams even after an error (no copy may outlive the call)
  const cudaError_t e1 = cudaStreamSynchronize(c.h2d), e2 = cudaStreamSynchronize(c.d2h),
                    e3 = cudaStreamSynchronize(c.st);
  if (rc) return rc;
  CUDA_TRY(e1);
  CUDA_TRY(e2);
  CUDA_TRY(e3);
  if (rep) {  // the model of what ran: wavefront phases on pw's row blocks, the middle on p's
    const int64_t mA = std::max<int64_t>(1, std::min(m, passes));
    const int64_t mC = std::min<int64_t>(m, passes - mA);
    const int64_t sA = std::min<int64_t>(total_steps, mA * p.h);
    const int64_t sC = mC ? total_steps - (passes - mC) * p.h : 0;
    const int64_t sB = total_steps - sA - sC;
    memset(rep, 0, sizeof *rep);
    const struct { const Plan* plan; int64_t steps; } parts[3] = {{&pw, sA}, {&p, sB}, {&pw, sC}};
    for (const auto& part : parts) {
      if (part.steps <= 0) continue;
      dtb_report r;
      fill_report<T>(*part.plan, nx, ny, part.steps, false, nullptr, &r);
      rep->global_load_cells += r.global_load_cells;
      rep->global_store_cells += r.global_store_cells;
      rep->halo_exchanged_cells += r.halo_exchanged_cells;
      rep->redundant_compute_cells += r.redundant_compute_cells;
      rep->useful_compute_cells += r.useful_compute_cells;
      rep->scratchpad_peak_bytes = r.scratchpad_peak_bytes;
      rep->elem_bytes = r.elem_bytes;
    }
  }
  if (cnt && rep) {
    unsigned long long h[8];
    CUDA_TRY(cudaMemcpy(h, cnt, sizeof h, cudaMemcpyDeviceToHost));
    rep->global_load_cells = (int64_t)h[0];
    rep->global_store_cells = (int64_t)h[1];
    rep->halo_exchanged_cells = (int64_t)h[2];
    rep->redundant_compute_cells = (int64_t)h[3] - nx * ny * total_steps;
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
  double wd[5];
  for (int i = 0; i < 5; ++i) wd[i] = (double)w[i];
  int rc = validate(nx, ny, pitch, wd, total_steps,
                    (flags & DTB_FLAG_FORCE_DEPTH) ? 1 : t_depth, valid);
  if (rc) return rc;
  if (n_gpus > 1) {
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
  if (!valid || (valid->x0 == 0 && valid->y0 == 0 && valid->width == nx && valid->height == ny)) {
    rc = solve_host_wave<T>(in, out, nx, ny, pitch, w, total_steps, flags, rep);
    if (rc >= 0) return rc;
  }
  int device;
  CUDA_TRY(cudaGetDevice(&device));
  // device copy with a 128-byte-multiple pitch: 16-byte aligned tile copies
  const int64_t dpitch = (nx + 2 + 31) / 32 * 32;
  const size_t bytes = (size_t)(ny + 2) * dpitch * sizeof(T);
  void* io = nullptr;
  if ((rc = arena_get(kArenaIo, device, 2 * bytes, &io))) return rc;
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

void reset_call_state() {
  g_err.clear();
  g_min_bytes = 0;
}

// one epoch of a multi-process slab with the fused halo stores (HaloMirror)
template <typename T>
int solve_dev_mirror(const T* d_in, T* d_out, int64_t nx, int64_t ny, int64_t pitch,
                     const T w[5], int64_t total_steps, const dtb_halo_mirror* mir,
                     cudaStream_t st, dtb_report* rep) {
  if (!mir) return fail(DTB_EINVAL, "null halo mirror");
  HaloMirror<T> m;
  for (int i = 0; i < 2; ++i) {
    m.peer[i] = static_cast<T*>(mir->peer[i]);
    m.r0[i] = mir->r0[i];
    m.r1[i] = mir->r1[i];
    m.p0[i] = mir->p0[i];
    if (m.peer[i] && (m.r0[i] < 0 || m.r1[i] > ny + 2 || m.r0[i] > m.r1[i] || m.p0[i] < 0))
      return fail(DTB_ERANGE, "halo mirror %d rows [%lld, %lld) -> %lld outside the grid", i,
                  (long long)m.r0[i], (long long)m.r1[i], (long long)m.p0[i]);
    if (!m.peer[i]) m.r0[i] = m.r1[i] = 0;
  }
  m.sw0 = mir->sw0;
  m.sw1 = mir->sw1;
  struct MirrorScope {
    explicit MirrorScope(const void* p) { g_halo_mirror = p; }
    ~MirrorScope() { g_halo_mirror = nullptr; }
  } scope(&m);
  return solve_dev<T>(d_in, d_out, nx, ny, pitch, w, total_steps, 1, nullptr,
                      DTB_FLAG_FORCE_PIPE, st, rep);
}

}  // namespace

extern "C" {

int dtb_j2d5pt_f64(const double* in, double* out, int64_t nx, int64_t ny, int64_t pitch,
                   const double w[5], int64_t total_steps, int64_t t_depth,
                   const dtb_rect* valid, int ilp, int n_gpus, unsigned flags,
                   dtb_report* rep) {
  reset_call_state();
  return solve_host<double>(in, out, nx, ny, pitch, w, total_steps, t_depth, valid, ilp, n_gpus,
                            flags, rep);
}

int dtb_j2d5pt_f32(const float* in, float* out, int64_t nx, int64_t ny, int64_t pitch,
                   const float w[5], int64_t total_steps, int64_t t_depth,
                   const dtb_rect* valid, int ilp, int n_gpus, unsigned flags,
                   dtb_report* rep) {
  reset_call_state();
  return solve_host<float>(in, out, nx, ny, pitch, w, total_steps, t_depth, valid, ilp, n_gpus,
                           flags, rep);
}

int dtb_j2d5pt_f64_dev(const double* d_in, double* d_out, int64_t nx, int64_t ny,
                       int64_t pitch, const double w[5], int64_t total_steps,
                       int64_t t_depth, const dtb_rect* valid, unsigned flags,
                       void* stream, dtb_report* rep) {
  reset_call_state();
  return solve_dev<double>(d_in, d_out, nx, ny, pitch, w, total_steps, t_depth, valid, flags,
                           (cudaStream_t)stream, rep);
}

int dtb_j2d5pt_f32_dev(const float* d_in, float* d_out, int64_t nx, int64_t ny,
                       int64_t pitch, const float w[5], int64_t total_steps,
                       int64_t t_depth, const dtb_rect* valid, unsigned flags,
                       void* stream, dtb_report* rep) {
  reset_call_state();
  return solve_dev<float>(d_in, d_out, nx, ny, pitch, w, total_steps, t_depth, valid, flags,
                          (cudaStream_t)stream, rep);
}

int dtb_plan(int64_t nx, int64_t ny, int32_t elem_bytes, int64_t total_steps, int64_t t_depth,
             unsigned flags, dtb_plan_info* out) {
  reset_call_state();
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
  const int depth = (flags & DTB_FLAG_FORCE_DEPTH) ? (int)t_depth : 0;
  Plan p;
  char err[512];
  int64_t min_bytes = 0;
  if (!make_plan(nx, ny, elem_bytes, total_steps, dev, force_mode(flags), depth, p, err,
                 sizeof err, &min_bytes))
    return plan_fail(err, min_bytes);
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

int dtb_j2d5pt_f64_dev_mirror(const double* d_in, double* d_out, int64_t nx, int64_t ny,
                              int64_t pitch, const double w[5], int64_t total_steps,
                              const dtb_halo_mirror* mir, void* stream, dtb_report* rep) {
  reset_call_state();
  return solve_dev_mirror<double>(d_in, d_out, nx, ny, pitch, w, total_steps, mir,
                                  (cudaStream_t)stream, rep);
}

int dtb_j2d5pt_f32_dev_mirror(const float* d_in, float* d_out, int64_t nx, int64_t ny,
                              int64_t pitch, const float w[5], int64_t total_steps,
                              const dtb_halo_mirror* mir, void* stream, dtb_report* rep) {
  reset_call_state();
  return solve_dev_mirror<float>(d_in, d_out, nx, ny, pitch, w, total_steps, mir,
                                 (cudaStream_t)stream, rep);
}

int dtb_ipc_malloc(int64_t bytes, void** ptr, uint8_t handle[64]) {
  reset_call_state();
  if (!ptr || !handle || bytes < 1) return fail(DTB_EINVAL, "bad ipc allocation request");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  void* p = nullptr;
  CUDA_TRY(cudaMalloc(&p, (size_t)bytes));
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    CUDA_TRY(e);
  }
  memcpy(handle, &h, 64);
  *ptr = p;
  return DTB_OK;
}

int dtb_ipc_free(void* ptr) {
  reset_call_state();
  CUDA_TRY(cudaFree(ptr));
  return DTB_OK;
}

int dtb_ipc_open(const uint8_t handle[64], void** ptr) {
  reset_call_state();
  if (!ptr || !handle) return fail(DTB_EINVAL, "null ipc handle");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  CUDA_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return DTB_OK;
}

int dtb_ipc_close(void* ptr) {
  reset_call_state();
  CUDA_TRY(cudaIpcCloseMemHandle(ptr));
  return DTB_OK;
}

int dtb_ipc_event_create(void** event, uint8_t handle[64]) {
  reset_call_state();
  if (!event || !handle) return fail(DTB_EINVAL, "null event output");
  static_assert(sizeof(cudaIpcEventHandle_t) == 64, "IPC event handle size");
  cudaEvent_t ev;
  CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming | cudaEventInterprocess));
  cudaIpcEventHandle_t h;
  const cudaError_t e = cudaIpcGetEventHandle(&h, ev);
  if (e != cudaSuccess) {
    cudaEventDestroy(ev);
    CUDA_TRY(e);
  }
  memcpy(handle, &h, 64);
  *event = ev;
  return DTB_OK;
}

int dtb_ipc_event_open(const uint8_t handle[64], void** event) {
  reset_call_state();
  if (!event || !handle) return fail(DTB_EINVAL, "null event handle");
  cudaIpcEventHandle_t h;
  memcpy(&h, handle, 64);
  cudaEvent_t ev;
  CUDA_TRY(cudaIpcOpenEventHandle(&ev, h));
  *event = ev;
  return DTB_OK;
}

int dtb_event_destroy(void* event) {
  reset_call_state();
  CUDA_TRY(cudaEventDestroy((cudaEvent_t)event));
  return DTB_OK;
}

int dtb_event_record(void* event, void* stream) {
  reset_call_state();
  CUDA_TRY(cudaEventRecord((cudaEvent_t)event, (cudaStream_t)stream));
  return DTB_OK;
}

int dtb_stream_wait_event(void* stream, void* event) {
  reset_call_state();
  CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, (cudaEvent_t)event, 0));
  return DTB_OK;
}

int64_t dtb_last_launch_count(void) { return g_launches; }

int64_t dtb_last_min_required_bytes(void) { return g_min_bytes; }

int64_t dtb_last_trace(int64_t* out, int64_t n) {
  const int64_t m = std::min<int64_t>(n, (int64_t)g_trace.size());
  for (int64_t i = 0; i < m && out; ++i) out[i] = g_trace[(size_t)i];
  return (int64_t)g_trace.size() / 8;
}

int dtb_device_info(int32_t* sms, int64_t* smem_optin_per_block, int64_t* l2_bytes,
                    int32_t* cc_major, int32_t* cc_minor) {
  reset_call_state();
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
  reset_call_state();
  if (nx < 1 || ny < 1 || pitch < nx + 2) return fail(DTB_EINVAL, "bad fill dims");
  return launch_fill<double>(d_out, pitch, (int)nx, (int)ny, seed, ghost, 0, ny + 2,
                             (cudaStream_t)stream);
}

int dtb_fill_random_f32(float* d_out, int64_t nx, int64_t ny, int64_t pitch, uint64_t seed,
                        double ghost, void* stream) {
  reset_call_state();
  if (nx < 1 || ny < 1 || pitch < nx + 2) return fail(DTB_EINVAL, "bad fill dims");
  return launch_fill<float>(d_out, pitch, (int)nx, (int)ny, seed, ghost, 0, ny + 2,
                            (cudaStream_t)stream);
}

int dtb_fill_random_rows_f64(double* d_out, int64_t nx, int64_t ny, int64_t pitch, uint64_t seed,
                             double ghost, int64_t row0, int64_t nrows, void* stream) {
  reset_call_state();
  if (nx < 1 || ny < 1 || pitch < nx + 2 || row0 < 0 || nrows < 0 || row0 + nrows > ny + 2)
    return fail(DTB_EINVAL, "bad fill rows");
  return launch_fill<double>(d_out, pitch, (int)nx, (int)ny, seed, ghost, row0, nrows,
                             (cudaStream_t)stream);
}

const char* dtb_last_error(void) { return g_err.c_str(); }

}  // extern "C"
