// dtb_plan.h — the B200 tile planner (host C++).
//
// Replaces the reference's capacity planner (planner.py:151-243) for the
// B200 execution. The reference models each SM ("worker") as holding a
// double-buffered column slice of one serially-processed tile
// (footprint 2*(ceil(w/workers)+2)*h*elem, planner.py:151-169). On B200 the
// unit is a CTA with a single-buffered, in-place smem tile:
//   footprint = load_h * (32*K) * elem            (one copy, fixed lane pitch)
// and tiles are 2-D so that a temporal halo of depth h costs O(h/edge) extra
// work instead of the reference's full-width row bands (planner.py:230-231).
//
// Two execution modes:
//   resident  — one persistent CTA per SM, the whole domain lives in smem for
//               the whole solve; halos of depth h are exchanged through L2 with
//               per-CTA epoch flags every h steps (no grid-wide barrier);
//   streaming — domains larger than aggregate smem: every pass loads each tile
//               (owned + h halo) from HBM, fuses h steps in smem, stores the
//               owned cells; passes ping-pong between two HBM buffers.
// The cost model below scores candidates in SM clock cycles per time step
// using the measured B200 rates (profiles/r01_microbench_peaks.log): 64 FP64 /
// 128 FP32 lanes per SM per clock, 9 separately-rounded ops per cell update.
#pragma once
#include <stdint.h>
#include <vector>

namespace dtb {

struct Split {
  int n = 0;
  std::vector<int> o0, o1;  // owned [o0, o1) in interior coordinates
  std::vector<int> l0, l1;  // load  [l0, l1), within [-1, N+1)
  int max_load = 0;
  bool dyn = false;         // some load width not a multiple of the lane width
};

struct DevInfo {
  int sms = 148;
  int64_t smem_optin = 232448;
  int64_t l2_bytes = 126 * 1024 * 1024;
  int64_t smem_per_sm = 233472;
};

struct Plan {
  int mode = 0;  // 0 resident, 1 streaming (tile sweep), 2 naive, 3 pipelined streaming
  int elem = 8;
  int K = 4;
  int warps = 16;
  int h = 4;
  Split sx, sy;
  int ctas = 0;
  int ctas_per_sm = 1;
  int64_t smem_bytes = 0;
  double cycles_per_step = 0;  // cost model
  double cells_per_clk = 0;
  int64_t computed_cells_per_step = 0;
  bool dyn() const { return sx.dyn; }
};

// Split [0, N) into n tiles of roughly equal LOAD extent, halo depth h,
// lane alignment `align` (load extents made multiples of it by growing the
// halo into the neighbour, never past the ghost ring). Returns false if some
// load extent exceeds maxL or a tile owns fewer than min_owned cells.
// `align`/`off`: load extents are grown (when the neighbour has the cells)
// to L = off (mod align); a miss is allowed in y (off != 0), flagged dyn in x.
// `start_align` > 1: interior boundaries are nudged so every load region
// starts at a padded index divisible by it (16-byte aligned tile copies).
bool make_split(int N, int n, int h, int align, int maxL, int min_owned, Split& s,
                int off = 0, int start_align = 1, int spread = 1);

// Choose the execution plan. force: 0 auto, 1 streaming, 2 naive, 3 pipelined,
// 4 resident. depth > 0 pins the halo depth. On failure, err holds the message
// and *min_bytes (if non-null) the smallest per-CTA shared memory a plan of the
// requested kind would need.
bool make_plan(int64_t nx, int64_t ny, int elem, int64_t steps, const DevInfo& dev,
               int force, int depth, Plan& out, char* err, int errlen,
               int64_t* min_bytes = nullptr);

}  // namespace dtb
