// dtb_plan.cpp — B200 tile planner; see dtb_plan.h for the model.
#include "dtb_plan.h"

#include <algorithm>
#include <mutex>
#include <string>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace dtb {

bool make_split(int N, int n, int h, int align, int maxL, int min_owned, Split& s, int off,
                int start_align, int spread) {
  s = Split();
  if (n < 1 || N < 1) return false;
  s.n = n;
  s.o0.resize(n); s.o1.resize(n); s.l0.resize(n); s.l1.resize(n);
  std::vector<int> left(n), right(n);
  long S = N;
  for (int i = 0; i < n; ++i) {
    left[i] = (i == 0) ? 1 : h;
    right[i] = (i == n - 1) ? 1 : h;
    S += left[i] + right[i];
  }
  // equal load extents: the per-CTA cost is set by the load region
  const long Lt = S / n, rem = S % n;
  int x = 0;
  for (int i = 0; i < n; ++i) {
    // spread == 2: the +1 remainder rows go to even tiles first (CTA pairs)
    const long rank = spread == 2 ? ((i & 1) ? (n + 1) / 2 + i / 2 : i / 2) : i;
    long own = Lt + (rank < rem ? 1 : 0) - left[i] - right[i];
    if (own < std::max(1, min_owned)) return false;
    s.o0[i] = x;
    s.o1[i] = x + (int)own;
    x += (int)own;
  }
  if (x != N) return false;
  if (start_align > 1) {
    // move interior boundaries so each load region starts on a 16-byte chunk
    // of the padded row (padded index l0 + 1 = o0 - h + 1 divisible):
    // whole-chunk cp.async / vector stores for the tile copies
    for (int i = 1; i < n; ++i) {
      const int b = s.o0[i];
      const int r = ((b - h + 1) % start_align + start_align) % start_align;
      const int nb = (r * 2 <= start_align) ? b - r : b + (start_align - r);
      if (nb - s.o0[i - 1] >= std::max(1, min_owned) && s.o1[i] - nb >= std::max(1, min_owned)) {
        s.o1[i - 1] = nb;
        s.o0[i] = nb;
      }
    }
  }
  for (int i = 0; i < n; ++i) {
    s.l0[i] = std::max(s.o0[i] - left[i], -1);
    s.l1[i] = std::min(s.o1[i] + right[i], N + 1);
  }
  for (int i = 0; i < n; ++i) {
    int L = s.l1[i] - s.l0[i];
    int ext = ((off - L) % align + align) % align;
    if (ext && L + ext > maxL) ext = 0;  // keep within capacity (y: best effort)
    if (ext) {
      // grow the halo into a neighbour (never beyond that neighbour's owned cells)
      int rlim = (i + 1 < n) ? s.o1[i + 1] : N + 1;
      int take = std::max(0, std::min(ext, rlim - s.l1[i]));
      s.l1[i] += take;
      ext -= take;
      int llim = (i > 0) ? s.o0[i - 1] : -1;
      take = std::max(0, std::min(ext, s.l0[i] - llim));
      s.l0[i] -= take;
      ext -= take;
      if (ext && off == 0) s.dyn = true;
    }
    s.max_load = std::max(s.max_load, s.l1[i] - s.l0[i]);
  }
  return s.max_load <= maxL;
}

namespace {

struct Shape { int K; int warps; };

// dtb_pipe.cuh kPipeWarps / kPipeStages / PipeCfg
constexpr int kPlanPipeStages = 4;
// lane width and warps per CTA of the pipe kernel per element size (PipeCfg)
constexpr int plan_pipe_K(int elem) { return elem == 8 ? 4 : 8; }
constexpr int plan_pipe_warps(int) { return 16; }

// kernel shapes compiled into libdtb_b200.so (dtb_resident.cuh / dtb_stream.cu):
// 32 B of row state per lane (fp64 K=4, fp32 K=8: one 1 KB smem row per
// warp-row), 8 warps
std::vector<Shape> shapes_for(int elem) {
  if (elem == 8) return {{4, 8}};
  return {{8, 8}};
}

std::vector<int> depths_for(int depth) {
  std::vector<int> v;
  if (depth > 0) v.push_back(depth);
  else for (int h = 2; h <= 32; h += 2) v.push_back(h);
  return v;
}

double lanes_per_clk(int elem) { return elem == 8 ? 64.0 : 128.0; }
// FP32 is issue-bound (FADD/FMUL alone fill the 4 issue slots per SM per
// clock), so the non-FP instructions per row cost throughput there.
double fp_efficiency(int elem) { return elem == 8 ? 0.92 : 0.80; }

// Band heights exactly as the kernel splits them (dtb_core.cuh band_rows).
static void band_heights(int rows, int nb, std::vector<int>& hts) {
  hts.assign(nb, 0);
  for (int b = 0; b < nb; ++b) hts[b] = rows / nb + (b < rows % nb ? 1 : 0);
}

// SM cycles for one CTA to advance a (Lw x Lh) tile by `steps` steps. Warp w
// runs on sub-partition w % 4; a sweep lasts as long as the busiest
// sub-partition's FP work (16 FP64 / 32 FP32 lanes per SMSP per clock).
double tile_cycles(int elem, int K, int warps, int Lh, int steps) {
  const int rows = Lh - 2;
  if (rows <= 0 || steps <= 0) return 0;
  const double lane_rate = lanes_per_clk(elem) / 4.0 * fp_efficiency(elem);
  const double row_cost = 32.0 * K * 9.0 / lane_rate;  // one warp-row on one SMSP
  double cyc = 0;
  int s = steps;
  std::vector<int> hts;
  if (s >= 2 && rows >= 2) {
    const int nb = std::max(1, std::min(warps, rows / 2));
    band_heights(rows, nb, hts);
    double smsp[4] = {0, 0, 0, 0};
    for (int b = 0; b < nb; ++b) smsp[b % 4] += (2.0 * hts[b] + 2.0) * row_cost;
    const double sweep = *std::max_element(smsp, smsp + 4) + 400.0;  // + barriers, fill
    cyc += (s / 2) * sweep;
    s %= 2;
  }
  if (s) {
    const int nb = std::max(1, std::min(warps, rows));
    band_heights(rows, nb, hts);
    double smsp[4] = {0, 0, 0, 0};
    for (int b = 0; b < nb; ++b) smsp[b % 4] += hts[b] * row_cost * 1.25;
    cyc += s * (*std::max_element(smsp, smsp + 4) + 300.0);
  }
  return cyc;
}

// sustained HBM bytes per SM clock (6545 GB/s measured copy, ~1.9 GHz)
constexpr double kHbmBytesPerClk = 3400.0;
// L2 bytes per clock for the resident halo exchange and epoch handshake
constexpr double kL2BytesPerClk = 5000.0;
constexpr double kExchangeLatency = 3500.0;  // flag publish + neighbour poll (~2 x 0.48 us)

bool plan_resident(int64_t nx, int64_t ny, int elem, int64_t steps, const DevInfo& dev,
                   int depth, Plan& best) {
  bool found = false;
  const char* mt = getenv("DTB_MAX_TILES");  // experiments: cap the resident tile count
  const int max_tiles = mt ? atoi(mt) : 1 << 30;
  const char* ya = getenv("DTB_YALIGN");  // experiments: load-height alignment (rows - 2)
  const int yalign_env = ya ? atoi(ya) : 0;
  for (const Shape& sh : shapes_for(elem)) {
    const int K = sh.K, W = sh.warps;
    const int Lw_max = 32 * K;
    const int64_t row_bytes = (int64_t)Lw_max * elem;
    const int maxRows = (int)((dev.smem_optin - 1024) / row_bytes);
    if (maxRows < 3) continue;
    // no load-height padding: the band sweeps take any row count (padding
    // rows-2 to a multiple of 4 bands x 8 rows cost C2 6 % and C3a 11 %)
    const int yalign = yalign_env > 0 ? yalign_env : 1;
    for (int h : depths_for(depth)) {
      const int hh = (int)std::min<int64_t>(h, std::max<int64_t>(steps, 1));
      const int ntx_min = (int)((nx + 2 + Lw_max - 1) / Lw_max);
      for (int ntx = std::max(1, ntx_min); ntx <= std::min<int64_t>(dev.sms, nx); ++ntx) {
        Split sx;
        if (!make_split((int)nx, ntx, h, K, Lw_max, ntx > 1 ? h : 1, sx, 0, 16 / elem)) continue;
        const int nty_max = (int)std::min<int64_t>(dev.sms / ntx, ny);
        const int nty_lo = std::max(1, nty_max - 2);
        for (int nty = nty_max; nty >= nty_lo; --nty) {
          if (ntx * nty > max_tiles) continue;
          Split sy;
          if (!make_split((int)ny, nty, h, yalign, maxRows, nty > 1 ? h : 1, sy, 2)) continue;
          // cost per epoch of hh steps: slowest CTA + exchange
          double cyc = tile_cycles(elem, K, W, sy.max_load, hh);
          if (steps > hh) {
            const double band = 2.0 * h * (sx.max_load + sy.max_load) * elem;  // write + read
            cyc += kExchangeLatency + 2.0 * band * dev.sms / kL2BytesPerClk;
          }
          const double per_step = cyc / hh;
          const double cpc = (double)nx * ny / per_step;
          if (!found || cpc > best.cells_per_clk) {
            found = true;
            best.mode = 0;
            best.elem = elem;
            best.K = K;
            best.warps = W;
            best.h = h;
            best.sx = sx;
            best.sy = sy;
            best.ctas = ntx * nty;
            best.ctas_per_sm = 1;
            best.smem_bytes = (int64_t)sy.max_load * row_bytes;
            best.cycles_per_step = per_step;
            best.cells_per_clk = cpc;
          }
        }
        if (sx.max_load < Lw_max / 2 && ntx > ntx_min) break;
      }
    }
  }
  return found;
}

bool plan_streaming(int64_t nx, int64_t ny, int elem, int64_t steps, const DevInfo& dev,
                    int depth, Plan& best) {
  bool found = false;
  for (const Shape& sh : shapes_for(elem)) {
    const int K = sh.K, W = sh.warps;
    const int Lw_max = 32 * K;
    const int64_t row_bytes = (int64_t)Lw_max * elem;
    for (int occ = 1; occ <= 2; ++occ) {  // occ = tile buffers per CTA (2: double-buffered)
      const int64_t smem_cta = (dev.smem_optin - 1024) / occ;
      const int maxRows = (int)(smem_cta / row_bytes);
      if (maxRows < 8) continue;
      for (int h : depths_for(depth)) {
        const int hh = (int)std::min<int64_t>(h, std::max<int64_t>(steps, 1));
        // interior tiles own at most Lw_max - 2h columns
        const int per = std::max(1, Lw_max - 2 * h);
        const int ntx_min = (int)std::max<int64_t>(1, std::max<int64_t>(
            (nx + 2 + Lw_max - 1) / Lw_max, (nx + per - 1) / per - 1));
        for (int ntx = ntx_min; ntx <= ntx_min + 3 && ntx <= nx; ++ntx) {
          Split sx;
          if (!make_split((int)nx, ntx, h, K, Lw_max, 1, sx, 0, 16 / elem)) continue;
          // tallest tiles that fit, and a few shorter ones (band balance)
          const int per_y = std::max(1, maxRows - 2 * h);
          int nty0 = (int)std::max<int64_t>(
              1, std::max<int64_t>((ny + 2 + maxRows - 1) / maxRows, (ny + per_y - 1) / per_y - 1));
          for (int nty = nty0; nty <= std::min<int64_t>(ny, nty0 + 8); ++nty) {
          Split sy;
          if (!make_split((int)ny, nty, h, 1, maxRows, 1, sy, 2)) continue;
          const int64_t ntiles = (int64_t)ntx * nty;
          const int64_t slots = dev.sms;  // one CTA per SM
          const double waves = std::ceil((double)ntiles / slots);
          const double tc = tile_cycles(elem, K, W, sy.max_load, hh);
          const double load_b = (double)sx.max_load * sy.max_load * elem;
          const double store_b = (double)(sx.max_load - 2 * h) * (sy.max_load - 2 * h) * elem;
          // per-tile memory time at this SM's share of HBM bandwidth
          const double mem_cta = (load_b + store_b) / (kHbmBytesPerClk / slots);
          // double-buffered: the next tile's load overlaps this tile's compute.
          // Calibrated on B200 (tools/sweep_bench.py DTB_TRACE=1, round 1): each
          // tile also pays ~10k cycles of copy issue, pipeline fill and band
          // prologue/epilogue, and the per-CTA copies reach ~half the share
          // of HBM bandwidth the model assumes.
          const double per_tile = (occ == 2 ? std::max(tc, 2.0 * mem_cta) : tc + 2.0 * mem_cta)
                                  + 10000.0;
          const double pass = waves * per_tile + mem_cta + 6000.0;
          const double per_step = pass / hh;
          const double cpc = (double)nx * ny / per_step;
          if (!found || cpc > best.cells_per_clk) {
            found = true;
            best.mode = 1;
            best.elem = elem;
            best.K = K;
            best.warps = W;
            best.h = h;
            best.sx = sx;
            best.sy = sy;
            best.ctas = (int)std::min<int64_t>(ntiles, slots);
            best.ctas_per_sm = occ;  // streaming: tile buffers per CTA
            best.smem_bytes = (int64_t)sy.max_load * row_bytes;
            best.cycles_per_step = per_step;
            best.cells_per_clk = cpc;
          }
          }
        }
      }
    }
  }
  return found;
}

// Pipelined streaming (dtb_pipe.cuh): S = 4 stage warps per pipeline, two
// pipelines per CTA, h = 8 steps per pass; tiles are column strips cut into
// a few long segments so that there are about two pipelines' worth of
// segments per SM.
bool plan_pipe(int64_t nx, int64_t ny, int elem, int64_t steps, const DevInfo& dev, Plan& best) {
  const int K = plan_pipe_K(elem), W = plan_pipe_warps(elem), S = kPlanPipeStages, P = W / S,
            h = 2 * S;
  const int Lw_max = 32 * K;
  const int per = Lw_max - 2 * h;
  Split sx;
  int ntx = (int)std::max<int64_t>(1, (nx + per - 1) / per - 1);
  for (; ntx <= nx; ++ntx)
    if (make_split((int)nx, ntx, h, K, Lw_max, 1, sx, 0, 16 / elem)) break;
  if (ntx > nx) return false;
  // segments per strip: every pipeline marches ceil(tiles / pipelines) tiles
  // (waves) of ~ny/nseg + 2h rows plus a pipeline fill; pick the count that
  // minimises that (one wave when the strips alone fill the device, several
  // shorter waves when they would leave SMs idle)
  const int64_t want = (int64_t)dev.sms * P;
  const int64_t seg_max = std::max<int64_t>(1, ny / (2 * h));
  int nseg = 0;
  double best_rows = 0;
  for (int64_t n = 1; n <= std::min<int64_t>(seg_max, 4 * want); ++n) {
    const int64_t waves = (ntx * n + want - 1) / want;
    const double rows = (double)waves * ((double)(ny + n - 1) / n + 2 * h + 4 * S);
    if (nseg == 0 || rows < best_rows * 0.999) {
      nseg = (int)n;
      best_rows = rows;
    }
  }
  Split sy;
  for (; nseg >= 1; --nseg)
    if (make_split((int)ny, nseg, h, 1, 1 << 30, nseg > 1 ? h : 1, sy)) break;
  if (nseg < 1) return false;
  best.mode = 3;
  best.elem = elem;
  best.K = K;
  best.warps = W;
  best.h = h;
  best.sx = sx;
  best.sy = sy;
  const int64_t ntiles = (int64_t)ntx * nseg;
  best.ctas = (int)std::min<int64_t>(dev.sms, (ntiles + P - 1) / P);
  best.ctas_per_sm = 1;
  // dtb_pipe.cuh PipeCfg: stage 0's prefetch ring is deeper for fp64
  const int ring = 12, ring0 = elem == 8 ? 16 : 12;
  best.smem_bytes = (int64_t)(ring0 + (S - 1) * ring) * Lw_max * elem * P;
  // cost: all lane-cells of every pass at ~70% of the FP issue rate + fill
  double lane_cells = 0;
  for (int i = 0; i < sx.n; ++i)
    for (int j = 0; j < sy.n; ++j)
      lane_cells += 32.0 * K * (sy.l1[j] - sy.l0[j]);
  // issue-efficiency calibrated on B200 (round 1: 16 warps, 4 pipelines/CTA)
  const double rate = (elem == 8 ? 64.0 * 0.49 : 128.0 * 0.37) / 9.0 * dev.sms;
  best.cycles_per_step = lane_cells / rate + 2000.0 / h;
  best.cells_per_clk = (double)nx * ny / best.cycles_per_step;
  (void)steps;
  return true;
}

}  // namespace

static bool make_plan_search(int64_t nx, int64_t ny, int elem, int64_t steps,
                             const DevInfo& dev, int force, int depth, Plan& out, char* err,
                             int errlen, int64_t* min_bytes);

// The planner's search (depths x tile counts x shapes) costs ~0.5 ms of host
// time; solves of the same shape reuse the last plans (small MRU cache).
bool make_plan(int64_t nx, int64_t ny, int elem, int64_t steps, const DevInfo& dev, int force,
               int depth, Plan& out, char* err, int errlen, int64_t* min_bytes) {
  struct Key {
    int64_t nx, ny, steps, smem_optin, l2, smem_sm;
    int elem, force, depth, sms, max_tiles;
    bool operator==(const Key& o) const {
      return nx == o.nx && ny == o.ny && steps == o.steps && smem_optin == o.smem_optin &&
             l2 == o.l2 && smem_sm == o.smem_sm && elem == o.elem && force == o.force &&
             depth == o.depth && sms == o.sms && max_tiles == o.max_tiles;
    }
  };
  static std::mutex mu;
  static std::vector<std::pair<Key, Plan>> cache;  // most recent first
  const char* mt = getenv("DTB_MAX_TILES");
  const Key key{nx, ny, steps, dev.smem_optin, dev.l2_bytes, dev.smem_per_sm,
                elem, force, depth, dev.sms, mt ? atoi(mt) : 0};
  if (min_bytes) *min_bytes = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (size_t i = 0; i < cache.size(); ++i) {
      if (cache[i].first == key) {
        out = cache[i].second;
        if (i) std::rotate(cache.begin(), cache.begin() + i, cache.begin() + i + 1);
        return true;
      }
    }
  }
  if (!make_plan_search(nx, ny, elem, steps, dev, force, depth, out, err, errlen, min_bytes))
    return false;
  std::lock_guard<std::mutex> lk(mu);
  cache.insert(cache.begin(), {key, out});
  if (cache.size() > 32) cache.pop_back();
  return true;
}

// Smallest shared memory per CTA that could hold a plan of this kind: the
// streaming kernels need one tile of a single owned row plus its 2h halo rows
// (a full lane-width row each); a resident plan needs the whole domain spread
// over the device's CTAs with depth-h halos. Carried by
// InfeasiblePlanError.min_required_bytes (planner.py:51-56, 222-228).
static int64_t min_required_bytes(int64_t nx, int64_t ny, int elem, int h, const DevInfo& dev,
                                  bool resident) {
  const int K = elem == 8 ? 4 : 8;
  const int64_t row_bytes = 32LL * K * elem;
  if (!resident) return std::min<int64_t>(1 + 2LL * h, ny + 2) * row_bytes;
  const int64_t per = std::max<int64_t>(1, 32LL * K - 2LL * h);
  const int64_t ntx = std::max<int64_t>(1, (nx + per - 1) / per);
  const int64_t nty = std::max<int64_t>(1, dev.sms / ntx);
  const int64_t rows = (ny + 2 + 2LL * h * (nty - 1) + nty - 1) / nty;
  return rows * row_bytes;
}

static bool make_plan_search(int64_t nx, int64_t ny, int elem, int64_t steps,
                             const DevInfo& dev, int force, int depth, Plan& out, char* err,
                             int errlen, int64_t* min_bytes) {
  if (nx < 1 || ny < 1) {
    snprintf(err, errlen, "domain dims must be at least 1x1, got %lldx%lld", (long long)nx,
             (long long)ny);
    return false;
  }
  if (nx > (1 << 30) || ny > (1 << 30)) {
    snprintf(err, errlen, "domain %lldx%lld too large", (long long)nx, (long long)ny);
    return false;
  }
  Plan p;
  bool ok = false;
  if (force == 2) {
    p.mode = 2;
    p.elem = elem;
    p.h = 1;
    ok = true;
  } else if (force == 3) {
    ok = plan_pipe(nx, ny, elem, steps, dev, p);
  } else if (force == 4) {
    ok = plan_resident(nx, ny, elem, steps, dev, depth, p);
  } else if (force == 1) {
    ok = plan_streaming(nx, ny, elem, steps, dev, depth, p);
  } else {
    // auto: smem-resident when the grid fits aggregate smem; otherwise the
    // pipelined streaming kernel (measured faster than the tile-sweep
    // streaming kernel on B200: 0.85 vs 0.64 Tcells/s fp64 at 16384^2), with
    // the tile sweep as the fallback (a forced depth other than 8, tiny grids)
    ok = plan_resident(nx, ny, elem, steps, dev, depth, p);
    if (!ok && (depth == 0 || depth == 2 * kPlanPipeStages) && nx >= 64 && ny >= 64)
      ok = plan_pipe(nx, ny, elem, steps, dev, p);
    if (!ok) ok = plan_streaming(nx, ny, elem, steps, dev, depth, p);
  }
  if (!ok) {
    const int h = depth > 0 ? depth : 2;
    const int64_t need = min_required_bytes(nx, ny, elem, h, dev, force == 4);
    if (min_bytes) *min_bytes = need;
    snprintf(err, errlen,
             "no B200 tiling fits %lldx%lld (elem %d B, depth %d) in %lld B of shared memory per "
             "CTA: needs at least %lld B",
             (long long)nx, (long long)ny, elem, depth, (long long)dev.smem_optin, (long long)need);
    return false;
  }
  // lane-cells updated per step (every inner cell of every load region)
  int64_t computed = 0;
  if (p.mode == 2) {
    computed = nx * ny;
  } else {
    for (int i = 0; i < p.sx.n; ++i)
      for (int j = 0; j < p.sy.n; ++j)
        computed += (int64_t)(p.sx.l1[i] - p.sx.l0[i] - 2) * (p.sy.l1[j] - p.sy.l0[j] - 2);
  }
  p.computed_cells_per_step = computed;
  out = p;
  return true;
}

}  // namespace dtb
